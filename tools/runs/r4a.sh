mkdir -p gpurun_out
T=r4a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for K in X ACP_QRCP_G1; do
env $K=1 timeout 1800 python bench.py --config c4g_2d_16x16 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_$K.log 2>&1; echo "c4g $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$K.log | head -1)"
done
