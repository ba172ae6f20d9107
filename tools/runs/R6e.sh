# R6e: PCG node sweep with warm starts (ACP_PCG_SWEEP = nodes per group; 0 = one cold batch): step time and iteration counts
mkdir -p gpurun_out
T=R6e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c3g_2d_8x8 c2_1d_semiconductor; do
for SW in 0 1 2 3; do
  ACP_PCG_SWEEP=$SW ACP_PCG_ITERS_HIST=1 timeout 600 python bench.py --config $C --steps 2 --warmup 2 --skip-cpu > gpurun_out/${T}_${C}_sw$SW.log 2>&1; echo "$C sweep $SW rc $?"
  grep '^{' gpurun_out/${T}_${C}_sw$SW.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['n_mu'], d['value'])"
  grep "useful" gpurun_out/${T}_${C}_sw$SW.log | tail -12 | awk '{s+=$7} END {print "column-iterations (last lines):", s}'
done
done
for SW in 0 2 1 3 4; do
  ACP_PCG_SWEEP=$SW ACP_PCG_ITERS_HIST=1 timeout 600 python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_c4g_sw$SW.log 2>&1; echo "c4g sweep $SW rc $?"
  grep '^{' gpurun_out/${T}_c4g_sw$SW.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['n_mu'], d['value'])"
  grep "acp pcg iters" gpurun_out/${T}_c4g_sw$SW.log | tail -40 | grep -E "node|useful" | tail -16
done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "golden or end_to_end or chi0 or sharded or dyson" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
