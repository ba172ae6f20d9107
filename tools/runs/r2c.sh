mkdir -p gpurun_out
T=r2c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_SYNC_CHECK=1 ACP_PCG_NOGRAPH=1 timeout 1500 python bench.py --config c4g_2d_16x16 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench c4g rc $?"; grep -o "AcpError.*" gpurun_out/${T}_bench.log | head -2
