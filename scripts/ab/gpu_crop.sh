# A/B: window kernel with per-view row-cropped boxes (KATS_BP_CROP=1, default) vs full-column boxes; parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/crop_test.log 2>&1; echo rc=$? >> gpurun_out/crop_test.log
for cfg in C5 C2 C5 C2; do
  for c in 1 0; do
    echo "$cfg crop=$c $(KATS_BP_CROP=$c timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3))')"
  done
done
timeout 120 python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/crop_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_bp_window$" -s 0 -c 1 -o gpurun_out/k5c5_crop -f python scripts/prof_step.py --config C5 --reps 1 >> gpurun_out/crop_prof.log 2>&1
