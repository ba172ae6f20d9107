mkdir -p gpurun_out
T=r1r
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_DEBUG= timeout 1500 python bench.py --config c3g_2d_8x8 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_c3g.log 2>&1; echo "bench c3g rc $?"; tail -c 2500 gpurun_out/${T}_bench_c3g.log
