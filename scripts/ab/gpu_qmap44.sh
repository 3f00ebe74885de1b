# A/B: TMEM kernel lane map 4x2 quarter / 4x4 half-warps (KATS_BP_QMAP=44) vs 8x1 / 8x2; parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
KATS_BP_QMAP=44 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/q44_test.log 2>&1; echo rc=$? >> gpurun_out/q44_test.log
for r in 1 2; do
  for cfg in C4 C3 C2; do
    for q in 44 0; do
      echo "$cfg qmap=$q $(KATS_BP_QMAP=$q timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3))')"
    done
  done
done
timeout 120 python scripts/prof_step.py --config C4 --pitches 8 --reps 1 > gpurun_out/q44_prof.log 2>&1 && \
KATS_BP_QMAP=44 ncu --set full --clock-control none --import-source on -k regex:"^k_bp_tmem$" -s 0 -c 1 -o gpurun_out/k5_q44 -f python scripts/prof_step.py --config C4 --pitches 8 --reps 1 >> gpurun_out/q44_prof.log 2>&1
