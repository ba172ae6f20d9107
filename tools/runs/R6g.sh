# R6g: golden parity margins (W sample per outer, D, lambda) of configs[2] / c3g for the node sweep variants
mkdir -p gpurun_out
T=R6g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
run() { env "$@" timeout 300 python tools/golden_margins.py $C 2>&1 | tail -1 | tee -a gpurun_out/${T}_margins.txt; }
C=c2_1d_semiconductor
run ACP_PCG_SWEEP=0
run ACP_PCG_SWEEP=2
run ACP_PCG_SWEEP=2 ACP_PCG_WARM_K=2
run ACP_PCG_SWEEP=2 ACP_PCG_WARM_K=4
run ACP_PCG_SWEEP=1 ACP_PCG_WARM_K=3
run ACP_PCG_SWEEP=2 ACP_PCG_WARM_TOL=0.01
run ACP_PCG_SWEEP=6
C=c3g_2d_8x8
run ACP_PCG_SWEEP=0
run ACP_PCG_SWEEP=1
