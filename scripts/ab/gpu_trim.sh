# A/B: TMEM kernel edge groups: pairs outside the warp union read a broadcast quad (KATS_BP_TRIM=1) vs their own
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
KATS_BP_TRIM=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/trim_test.log 2>&1; echo rc=$? >> gpurun_out/trim_test.log
for r in 1 2; do
  for cfg in C4 C3; do
    for t in 1 0; do
      echo "$cfg trim=$t $(KATS_BP_TRIM=$t timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3), "e2e", round(d["e2e"]["ms_per_step"],2))')"
    done
  done
done
timeout 120 python scripts/prof_step.py --config C4 --pitches 8 --reps 1 > gpurun_out/trim_prof.log 2>&1 && \
KATS_BP_TRIM=1 ncu --set full --clock-control none --import-source on -k regex:"^k_bp_tmem$" -s 0 -c 1 -o gpurun_out/k5_trim -f python scripts/prof_step.py --config C4 --pitches 8 --reps 1 >> gpurun_out/trim_prof.log 2>&1
