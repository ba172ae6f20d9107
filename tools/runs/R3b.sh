# Round 2, call R3b: step-time variance at c4g -- per-outer compress / chi0 / SMW event times over 6
# steps, with and without the nvidia-smi sampler
mkdir -p gpurun_out
T=${TAG:-R3b}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for V in smi nosmi; do
  if [ $V = nosmi ]; then export ACP_BENCH_NO_SMI=1; fi
  ACP_DYSON_PROF=1 timeout 1200 python bench.py --steps 6 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$V.log 2>gpurun_out/${T}_bench_$V.err; echo "bench $V rc $?"
  grep '^{' gpurun_out/${T}_bench_$V.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], d['e2e']['ms_each'], d['clocks'])"
  grep "dyson ms" gpurun_out/${T}_bench_$V.err
done
nvidia-smi -q -d PERFORMANCE,POWER,CLOCK | head -60 > gpurun_out/${T}_smi.txt
