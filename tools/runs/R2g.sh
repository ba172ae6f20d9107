mkdir -p gpurun_out
T=${TAG:-R2g}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for CN in "c3g_2d_8x8 7680" "c4g_2d_16x16 4096"; do
set -- $CN
ACP_F2C_PROF=1 timeout 300 python tools/k1_prof.py $1 $2 > gpurun_out/${T}_t.log 2>&1; grep f2c gpurun_out/${T}_t.log | tail -1; tail -1 gpurun_out/${T}_t.log | cut -c1-100
done
