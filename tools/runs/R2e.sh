mkdir -p gpurun_out
T=${TAG:-R2c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 3 > gpurun_out/${T}_t.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_f2c -s 3 -c 1 -o gpurun_out/${T}_prof_c4g -f \
    python tools/k1_time.py c4g_2d_16x16 4096 3 > gpurun_out/${T}_ncu_c4g.log 2>&1
echo "ncu c4g rc $?"; tail -2 gpurun_out/${T}_ncu_c4g.log
