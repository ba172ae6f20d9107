mkdir -p gpurun_out
T=r1zu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for cs in 0 4 6 8 12 16; do
  if [ $cs = 0 ]; then unset ACP_FFT2D_CS; else export ACP_FFT2D_CS=$cs; fi
  echo "cs=$cs $(timeout 300 python tools/k1_sweep.py c3g_2d_8x8 2048 2>&1 | tail -1)"
done
unset ACP_FFT2D_CS
timeout 600 python tools/k1_sweep.py c3g_2d_8x8 2048 > /dev/null 2>&1; echo "plain rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fft2d -s 2 -c 1 -o gpurun_out/${T}_fft2d \
    python tools/k1_sweep.py c3g_2d_8x8 2048 > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc $?"
