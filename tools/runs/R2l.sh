# Round 2, call l: c4g bench (default config) + launch list of one step (ncu, host-driven PCG loop)
mkdir -p gpurun_out
T=${TAG:-R2l}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1200 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep '^{' gpurun_out/${T}_bench.log | cut -c1-1500
ACP_PCG_HOSTLOOP=1 timeout 900 python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_plain.log 2>&1 && \
  ACP_PCG_HOSTLOOP=1 timeout 1500 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc $?"
