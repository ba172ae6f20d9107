#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, default bench (with cpu_baseline), reference arm,
# ncu launch list of one step (NVTX-filtered), ncu --set full of K1/K2/K3 at the bench shapes.
# Usage (under gpurun): bash tools/round_evidence.sh <tag> [main|full]
#   main: tests, smoke, bench, reference arm, ncu launch list;  full: ncu --set full captures
# (one ncu kind per gpurun call).
T=${1:-rX}
MODE=${2:-main}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
if [ "$MODE" = main ]; then
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc $?"; grep '^{' gpurun_out/${T}_bench.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo "ref rc $?"; grep '^{' gpurun_out/${T}_bench_ref.log | cut -c1-300
ACP_PCG_HOSTLOOP=1 timeout 600 python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_plain.log 2>&1 && \
  ACP_PCG_HOSTLOOP=1 timeout 900 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc $?"
else
for W in 0 1 2; do
  case $W in 0) K=k_fft1d;; 1) K=k_tn_cluster;; 2) K=k_pcg_update;; esac
  timeout 120 python profiles/kernel_probe.py --which $W > gpurun_out/${T}_probe$W.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/${T}_prof_$K -f \
      python profiles/kernel_probe.py --which $W > gpurun_out/${T}_ncu_full_$W.log 2>&1
  echo "ncu full $K rc $?"
done
fi
