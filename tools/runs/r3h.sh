mkdir -p gpurun_out
T=r3h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for r in 1 2 3; do
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "c1 rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
ACP_PCG_HOSTLOOP=1 timeout 600 python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_plain.log 2>&1; echo "plain rc $?"
ACP_PCG_HOSTLOOP=1 timeout 900 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc $?"
