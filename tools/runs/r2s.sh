mkdir -p gpurun_out
T=r2s
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "deferred" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
C=c3g_2d_8x8
ACP_PCG_HOSTLOOP=1 timeout 900 python bench.py --config $C --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_plain.log 2>&1; echo "plain rc $?"
ACP_PCG_HOSTLOOP=1 timeout 1800 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$C.csv \
    python bench.py --config $C --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_ncu_$C.log 2>&1
echo "launch list $C rc $?"
