mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r1f_build.log 2>&1 || { tail -20 gpurun_out/r1f_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r1f_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r1f_pytest.log
(timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 0,192,256; timeout 300 python tools/k1_sweep.py c2_1d_semiconductor 512 0,512,1024; timeout 300 python tools/k1_sweep.py c3_2d_8x8 512 0,288; timeout 300 python tools/k1_sweep.py c4_2d_16x16 256 0,512) > gpurun_out/r1f_k1sweep.log 2>&1; cat gpurun_out/r1f_k1sweep.log
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/r1f_bench.log 2>&1; echo "bench rc $?"; grep -o '"ms_per_step": [0-9.]*\|"K1_fourier_op": {[^}]*}' gpurun_out/r1f_bench.log
timeout 120 python tools/k1_sweep.py c1_1d_insulator 928 0 > /dev/null 2>&1 && timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_fft1d -s 5 -c 1 -f -o gpurun_out/r1f_k1_c1 python tools/k1_sweep.py c1_1d_insulator 928 0 > gpurun_out/r1f_ncu1.log 2>&1; echo "ncu1 rc $?"
