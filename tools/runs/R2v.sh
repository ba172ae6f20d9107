# Round 2, call v: c4g bench with per-pass times + kq per-phase profile; ncu --set full of K1/K2/K3
# at c4g (4096 columns, working set >> L2) for profiles/traffic.json
mkdir -p gpurun_out
T=${TAG:-R2v}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_KQ_PROF=1 timeout 1200 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>gpurun_out/${T}_bench.err; echo "bench rc $?"; grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], d['e2e'])"
grep kq gpurun_out/${T}_bench.err | sort | uniq -c | head
for w in 0 1 2; do
  timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 5 $w > gpurun_out/${T}_k$w.json 2>&1; echo "k$w rc $?"; cat gpurun_out/${T}_k$w.json | cut -c1-300
done
K=("k_f2c" "k_tn_cluster" "k_pcg_update_big")
for w in 0 1 2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K[$w]} -s 1 -c 1 -o gpurun_out/${T}_ncu_k$w \
    python tools/k1_time.py c4g_2d_16x16 4096 1 $w > gpurun_out/${T}_ncu_k$w.log 2>&1; echo "ncu k$w rc $?"
done
