# Round 2, call R3d: outer 1 of c4g shows PCG time 5-32 s (iteration counts vary between identical
# steps; once: no convergence in 2000 iterations).  Per-outer event times over 5 steps for: the fused
# 2D K1 as is, with cross-proxy fences, and the three-pass K1 (ACP_F2C=0).
mkdir -p gpurun_out
T=${TAG:-R3d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for V in "f2c" "pfence" "passes"; do
  case $V in f2c) E="";; pfence) E="ACP_F2C_PFENCE=1";; passes) E="ACP_F2C=0";; esac
  env $E ACP_DYSON_PROF=1 ACP_BENCH_NO_SMI=1 timeout 900 python bench.py --steps 5 --warmup 1 --skip-cpu > gpurun_out/${T}_$V.log 2>gpurun_out/${T}_$V.err; echo "$V rc $?"
  grep "dyson ms" gpurun_out/${T}_$V.err | cut -c45-
  grep "Error" gpurun_out/${T}_$V.err | tail -1
done
