# Round 2, call R4c: c4g with the PCG split into 2 / 3 node groups on their own streams (their K2/K3
# launches can share SMs out of phase) vs 1
mkdir -p gpurun_out
T=${TAG:-R4c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for G in 1 2 3; do
  ACP_PCG_GROUPS=$G ACP_DYSON_PROF=1 timeout 900 python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_g$G.log 2>gpurun_out/${T}_g$G.err; echo "groups $G rc $?"
  grep '^{' gpurun_out/${T}_g$G.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'])"
  grep "dyson ms" gpurun_out/${T}_g$G.err | tail -1
done
