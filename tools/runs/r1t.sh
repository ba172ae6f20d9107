mkdir -p gpurun_out
T=r1t
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_K1_PROFILE=1 timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 0 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep -o '"ms_per_step": [0-9.]*\|"K2_gemm_tn": {[^}]*}' gpurun_out/${T}_bench.log
(timeout 300 python tools/k1_sweep.py c3_2d_8x8 512 0,288; timeout 300 python tools/k1_sweep.py c4_2d_16x16 256 0,512) 2>&1 | grep config
