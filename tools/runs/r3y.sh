mkdir -p gpurun_out
T=r3y
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for S in 4 2 3 4 2 3; do
ACP_K2_ST32=$S timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "c1 st32=$S rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
for K in X ACP_K2_ST4; do
env $K=1 timeout 1800 python bench.py --config c4g_2d_16x16 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench4.log 2>&1; echo "c4g $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench4.log | head -1)"
done
