# TMEM kernel with 4x4 half-warps for single items (default) vs rows (KATS_BP_QMAP=0); C4 unchanged kernel
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/q44b_test.log 2>&1; echo rc=$? >> gpurun_out/q44b_test.log
for r in 1 2; do
  for cfg in C3 C4; do
    for q in 44 0; do
      echo "$cfg qmap=$q $(KATS_BP_QMAP=$q timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3), "e2e", round(d["e2e"]["ms_per_step"],2))')"
    done
  done
done
