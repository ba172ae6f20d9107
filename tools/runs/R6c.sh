# R6c: fused 2D K1 with consumed plane blocks discarded from L2 (discard.global.L2 after the TMA fetch): time,
# DRAM traffic and parity, against the default build path (ACP_F2C_DISCARD=0)
mkdir -p gpurun_out
T=R6c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for D in 0 1; do
  ACP_F2C_DISCARD=$D timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 0 2>&1 | tail -1 | tee -a gpurun_out/${T}_k1.txt
done
for SK in 14 16 24 30; do
  ACP_F2C_DISCARD=1 ACP_F2C_SKEW=$SK timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 0 2>&1 | tail -1 | tee -a gpurun_out/${T}_k1.txt
done
for D in 0 1; do
  ACP_F2C_DISCARD=$D timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_f2c -s 1 -c 1 \
    python tools/k1_time.py c4g_2d_16x16 38088 1 0 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/discard=$D /" | tee -a gpurun_out/${T}_k1.txt
done
ACP_F2C_DISCARD=1 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "f2c or fused or free_electron or fourier or golden" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
ACP_F2C_DISCARD=1 timeout 600 python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep '^{' gpurun_out/${T}_bench.log | cut -c1-330
