# R6h: node sweep at extrapolation order 3 (and 2): golden margins and step times vs the warm tolerance factor
mkdir -p gpurun_out
T=R6h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
run() { env "$@" timeout 300 python tools/golden_margins.py $C 2>&1 | tail -1 | tee -a gpurun_out/${T}_margins.txt; }
for C in c2_1d_semiconductor c3g_2d_8x8; do
run ACP_PCG_WARM_TOL=1.0
run ACP_PCG_WARM_TOL=0.1
run ACP_PCG_WARM_TOL=1.0 ACP_PCG_WARM_K=2
done
bench() { C=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 2 --warmup 2 --skip-cpu 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$C $*', d['ms_per_step'], d['value'])" | tee -a gpurun_out/${T}_times.txt; }
for C in c2_1d_semiconductor c3g_2d_8x8; do
bench $C ACP_PCG_WARM_TOL=1.0
bench $C ACP_PCG_WARM_TOL=0.1
bench $C ACP_PCG_WARM_TOL=1.0 ACP_PCG_SWEEP=1
bench $C ACP_PCG_WARM_TOL=1.0 ACP_PCG_SWEEP=2
done
bench c4g_2d_16x16 ACP_PCG_WARM_TOL=1.0
bench c4g_2d_16x16 ACP_PCG_WARM_TOL=0.1
bench c4g_2d_16x16 ACP_PCG_WARM_TOL=1.0 ACP_PCG_WARM_K=2
