mkdir -p gpurun_out
T=r1zc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c3_2d_8x8 c4_2d_16x16; do ACP_K1_PROFILE=1 timeout 300 python tools/k1_sweep.py $C 512 0 2>&1 | grep -E "phase|config"; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_fullsize.log 2>&1; echo "pytest fullsize rc $?"; tail -3 gpurun_out/${T}_pytest_fullsize.log
timeout 1500 python bench.py --config c2_1d_semiconductor --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c2.log 2>&1; echo "bench c2 rc $?"; grep '^{' gpurun_out/${T}_bench_c2.log | cut -c1-900
