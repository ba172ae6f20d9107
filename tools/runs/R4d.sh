# Round 2, call R4d: bench lines of the other configs on the final kernels (configs[2], c3g)
mkdir -p gpurun_out
T=${TAG:-R4d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c2_1d_semiconductor c3g_2d_8x8; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 > gpurun_out/${T}_bench_$C.log 2>&1; echo "$C rc $?"
  grep '^{' gpurun_out/${T}_bench_$C.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline'])"
done
