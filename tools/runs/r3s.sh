mkdir -p gpurun_out
T=r3s
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for O in 4 5; do ACP_F2_OCC=$O timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "2d_compiled" > gpurun_out/${T}_pytest$O.log 2>&1; echo "pytest occ$O rc $?"; done
for O in 3 4 5 3 4 5; do
ACP_F2_OCC=$O timeout 1500 python bench.py --config c3g_2d_8x8 --steps 2 --warmup 2 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "c3g occ=$O rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1) $(python -c "import json; d=json.loads(open('gpurun_out/${T}_bench.log').read().strip().splitlines()[-1]); print(round(d['kernels']['K1_fourier_op']['us'],1))")"
done
