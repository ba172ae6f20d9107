mkdir -p gpurun_out
T=r1zx
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for K in ACP_QRCP_GRID16 X ACP_QRCP_GRID16 X; do
env $K=1 timeout 900 python bench.py --config c2_1d_semiconductor --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$K.log 2>&1; echo "bench $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$K.log | head -1)"; grep -o "failed.*" gpurun_out/${T}_bench_$K.log | head -2
done
