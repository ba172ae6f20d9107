#!/bin/bash
# One GPU verification pass: parity tests, bench line, ncu launch list, ncu --set full on the hot kernels.
# Usage (under gpurun): bash tools/gpu_check.sh [tag] [config]
TAG=${1:-r1}
CFG=${2:-c1_1d_insulator}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc $?"; tail -c 3000 gpurun_out/${TAG}_bench.log
for C in ${PROBE2D:-}; do timeout 900 python tools/probe_2d.py $C 300 > gpurun_out/${TAG}_probe2d_$C.log 2>&1; echo "probe2d $C rc $?"; tail -3 gpurun_out/${TAG}_probe2d_$C.log; done
if [ "${SKIP_NCU:-0}" = "1" ]; then exit 0; fi
timeout 600 python bench.py --config $CFG --steps 1 --warmup 3 --skip-cpu > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --nvtx --nvtx-include "acp_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --config $CFG --steps 1 --warmup 3 --skip-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc $?"
for W in 0 1 2; do
  case $W in 0) K=k_fft1d;; 1) K=k_tn_cluster;; 2) K=k_pcg_update;; esac
  timeout 120 python profiles/kernel_probe.py --which $W --config $CFG > gpurun_out/${TAG}_probe$W.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/${TAG}_prof_$K -f \
      python profiles/kernel_probe.py --which $W --config $CFG > gpurun_out/${TAG}_ncu_full_$W.log 2>&1
  echo "ncu full $K rc $?"
done
