mkdir -p gpurun_out
T=r1zs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for combo in "X=1" "ACP_PCG_UNFUSED=1" "ACP_LU_SMEM_PANEL=1" "ACP_PCG_UNFUSED=1 ACP_LU_SMEM_PANEL=1"; do
env $combo timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1
echo "$combo: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
