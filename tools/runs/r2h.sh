mkdir -p gpurun_out
T=r2h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 300 python tools/qr_probe.py c1_1d_insulator gpurun_out/${T}_qrprof.txt 2>&1 | tail -3
