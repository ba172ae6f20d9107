mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r1c_build.log 2>&1 || { tail -20 gpurun_out/r1c_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r1c_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r1c_pytest.log
(timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 0,160,320,640,1024; timeout 300 python tools/k1_sweep.py c2_1d_semiconductor 512 0,256,512,1024; timeout 300 python tools/k1_sweep.py c3_2d_8x8 512 0,288,576,1024; timeout 300 python tools/k1_sweep.py c4_2d_16x16 256 0,512,1024) > gpurun_out/r1c_k1sweep.log 2>&1; cat gpurun_out/r1c_k1sweep.log
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/r1c_bench.log 2>&1; echo "bench rc $?"; grep -o '"ms_per_step": [0-9.]*\|"K1_fourier_op": {[^}]*}' gpurun_out/r1c_bench.log
for E in 1.0 0.3; do timeout 600 python tools/probe_2d.py c3_2d_8x8 300 $E 2>&1 | tail -1; done > gpurun_out/r1c_probe2d.log; cat gpurun_out/r1c_probe2d.log
timeout 900 python tools/probe_2d.py c4_2d_16x16 300 0.3 2>&1 | tail -1 >> gpurun_out/r1c_probe2d.log; tail -1 gpurun_out/r1c_probe2d.log
