mkdir -p gpurun_out
T=r2z
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c1_1d_insulator c2_1d_semiconductor c3g_2d_8x8 c4g_2d_16x16; do
S=3; [ $C = c4g_2d_16x16 ] && S=1
timeout 1800 python bench.py --config $C --steps $S --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1)"
done
