mkdir -p gpurun_out
T=r3t
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_F2_OCC=6 ACP_F2_OCC256=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "2d_compiled" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for O in 5 6 5 6; do
ACP_F2_OCC=$O timeout 1500 python bench.py --config c3g_2d_8x8 --steps 2 --warmup 2 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "c3g occ=$O rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
for O in 3 4; do
echo "c4g occ256=$O $(ACP_F2_OCC256=$O timeout 300 python tools/k1_sweep.py c4g_2d_16x16 4096 2>&1 | tail -1)"
done
for O in 3 4; do
echo "c4g occ256=$O $(ACP_F2_OCC256=$O timeout 300 python tools/k1_sweep.py c4g_2d_16x16 4096 2>&1 | tail -1)"
done
