mkdir -p gpurun_out
T=r2l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "chi0 or dyson or end_to_end" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
for C in c1_1d_insulator c2_1d_semiconductor; do
for G in 1 2 4 1 2 4; do
ACP_PCG_GROUPS=$G timeout 1500 python bench.py --config $C --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C G=$G rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1)"
done; done
