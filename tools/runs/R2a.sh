# Round 2, call a: FP64 peak microbenchmark + ncu --set full of the 2D K1 passes (c3g, c4g shapes).
mkdir -p gpurun_out
T=R2a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/micro/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/${T}_fp64_peak.txt 2>&1; echo "fp64 rc $?"; cat gpurun_out/${T}_fp64_peak.txt
for CN in "c3g_2d_8x8 7680" "c4g_2d_16x16 4096"; do
set -- $CN
timeout 300 python profiles/kernel_probe.py --which 0 --config $1 --ncols $2 > gpurun_out/${T}_probe_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_f2_ -s 3 -c 3 -o gpurun_out/${T}_prof_k1_$1 -f \
    python profiles/kernel_probe.py --which 0 --config $1 --ncols $2 > gpurun_out/${T}_ncu_$1.log 2>&1
echo "ncu $1 rc $?"; tail -3 gpurun_out/${T}_ncu_$1.log
done
