mkdir -p gpurun_out
T=r1zy
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for K in ACP_QRCP_GRID16 X ACP_QRCP_GRID16 ACP_QRCP_GRID16; do
env $K=1 timeout 900 python bench.py --config c2_1d_semiconductor --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$K.log 2>&1; echo "bench $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$K.log | head -1)"; grep -o "failed.*" gpurun_out/${T}_bench_$K.log | head -2
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_fullsize.py -k "free_electron and c2" -x -q > gpurun_out/${T}_memcheck.log 2>&1; echo "memcheck rc $?"; tail -5 gpurun_out/${T}_memcheck.log
