mkdir -p gpurun_out
T=r3p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c2_1d_semiconductor c3g_2d_8x8; do
ACP_PCG_HOSTLOOP=1 timeout 900 python bench.py --config $C --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_plain_$C.log 2>&1; echo "plain $C rc $?"
ACP_PCG_HOSTLOOP=1 timeout 1800 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$C.csv \
    python bench.py --config $C --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_ncu_$C.log 2>&1
echo "launch list $C rc $?"
done
