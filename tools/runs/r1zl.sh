mkdir -p gpurun_out
T=r1zl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
for C in c1_1d_insulator c2_1d_semiconductor c3g_2d_8x8; do
timeout 900 python bench.py --config $C --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C rc $?"
grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log
done
for C in c3g_2d_8x8 c2_1d_semiconductor; do
ACP_PCG_HOSTLOOP=1 timeout 1800 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$C.csv \
    python bench.py --config $C --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_ncu_$C.log 2>&1
echo "launch list $C rc $?"
done
