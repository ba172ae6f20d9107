# Round 2, call x: K3 A/B -- 64x64 tile (default) vs 128x64 XL tile (3 / 4 stages), EpBeta and EpAlpha,
# at c4g (N_occ 256, 4096 columns) and c2 (N_occ 128, 4096 columns); then c4g step time per variant
mkdir -p gpurun_out
T=${TAG:-R2x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c4g_2d_16x16 c2_1d_semiconductor; do
for X in 0 3 4; do for w in 2 3; do
  ACP_K3_XL=$X timeout 300 python tools/k1_time.py $C 4096 10 $w 2>&1 | tail -1 | cut -c1-200
done; done; done
for X in 0 3; do
  ACP_K3_XL=$X timeout 900 python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_xl$X.log 2>&1; echo "bench XL=$X rc $?"
  grep '^{' gpurun_out/${T}_bench_xl$X.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'])"
done
