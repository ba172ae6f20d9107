mkdir -p gpurun_out
T=r2m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 300 python tools/qr_probe.py c1_1d_insulator gpurun_out/${T}_qrprof.txt 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep -o "\"ms_per_step\": [0-9.]*" gpurun_out/${T}_bench.log | head -1
timeout 900 python -m pytest tests -q -m gpu -x -k "compress or qrcp or dyson or end_to_end" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
