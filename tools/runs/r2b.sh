mkdir -p gpurun_out
T=r2b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for K in ACP_FFT2D_CLUSTER X; do
env $K=1 timeout 1200 python bench.py --config c4g_2d_16x16 --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$K.log 2>&1; echo "bench c4g $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$K.log | head -1)"; grep -o "AcpError.*" gpurun_out/${T}_bench_$K.log | head -2
done
