mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r1d_build.log 2>&1 || { tail -20 gpurun_out/r1d_build.log; exit 1; }
(timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 0,96,128,160,192,256,320; timeout 300 python tools/k1_sweep.py c3_2d_8x8 512 0,192,288,384,576) > gpurun_out/r1d_k1sweep.log 2>&1; cat gpurun_out/r1d_k1sweep.log
timeout 120 python tools/k1_sweep.py c1_1d_insulator 928 160 > /dev/null 2>&1 && timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_fft1d -s 5 -c 1 -f -o gpurun_out/r1d_k1_c1 python tools/k1_sweep.py c1_1d_insulator 928 160 > gpurun_out/r1d_ncu1.log 2>&1; echo "ncu1 rc $?"
timeout 120 python tools/k1_sweep.py c3_2d_8x8 512 288 > /dev/null 2>&1 && timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_fft2d -s 5 -c 1 -f -o gpurun_out/r1d_k1_c3 python tools/k1_sweep.py c3_2d_8x8 512 288 > gpurun_out/r1d_ncu2.log 2>&1; echo "ncu2 rc $?"
