mkdir -p gpurun_out
T=r3d
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c3g_2d_8x8 c2_1d_semiconductor; do
for E in 0 1 2 0 1 2; do
ACP_K3_EPI=$E timeout 1500 python bench.py --config $C --steps 2 --warmup 2 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C EPI=$E rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1)"
done; done
