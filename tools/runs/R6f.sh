# R6f: node sweep with warm groups stopping at warm_tol * tol: golden parity margins and step times
mkdir -p gpurun_out
T=R6f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for F in 0.1 0.3; do
  ACP_PCG_WARM_TOL=$F timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "golden" > gpurun_out/${T}_golden_$F.log 2>&1; echo "golden warm_tol $F rc $?"; tail -3 gpurun_out/${T}_golden_$F.log; grep -E "^E +AssertionError" gpurun_out/${T}_golden_$F.log | head -5
done
for F in 0.1 0.3; do
  ACP_PCG_WARM_TOL=$F timeout 600 python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_c4g_$F.log 2>&1; echo "c4g warm_tol $F rc $?"
  grep '^{' gpurun_out/${T}_c4g_$F.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['n_mu'], d['value'])"
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest_gpu.log
for C in c3g_2d_8x8 c2_1d_semiconductor; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "$C rc $?"
  grep '^{' gpurun_out/${T}_bench_$C.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['n_mu'], d['value'])"
done
