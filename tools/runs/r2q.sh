mkdir -p gpurun_out
T=r2q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for G in 4 8 2 4 8; do
ACP_PCG_GROUPS=$G timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "c1 G=$G rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
ACP_PCG_GROUPS=8 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "chi0 or dyson" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest G8 rc $?"; tail -1 gpurun_out/${T}_pytest.log
