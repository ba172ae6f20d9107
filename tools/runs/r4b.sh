mkdir -p gpurun_out
T=r4b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for O in 0 5 8 0 5 8; do
ACP_K3_OCC=$O timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "c1 k3occ=$O rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
