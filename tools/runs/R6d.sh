# R6d: placement of the L2 discard of consumed K1 plane blocks (build-time -DACP_F2C_DISCARD=m): time + DRAM bytes
mkdir -p gpurun_out
T=R6d
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
P=paper_1605_08021_b200
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for M in 0 3 2 1 0; do
  nvcc $FL -DACP_F2C_DISCARD=$M -c $P/csrc/fft2c.cu -o $P/build/fft2c.o && nvcc -shared -gencode arch=compute_100a,code=sm_100a $P/build/*.o -o $P/libacp_b200.so -lcudart || { echo "build $M failed"; continue; }
  timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 5 0 2>&1 | tail -1 | sed "s/^/mode=$M /" | tee -a gpurun_out/${T}_k1.txt
  if [ $M != 0 ]; then
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_f2c -s 1 -c 1 \
    python tools/k1_time.py c4g_2d_16x16 38088 1 0 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/mode=$M /" | tee -a gpurun_out/${T}_k1.txt
  fi
done
