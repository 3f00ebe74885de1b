# A/B: window kernel with four items per CTA (KATS_BP_WINV=3, byte ring) vs two (default) at C5; parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
KATS_BP_WINV=3 timeout 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -k "c5 or C5 or batch" > gpurun_out/ni4_test.log 2>&1; echo rc=$? >> gpurun_out/ni4_test.log
for r in 1 2; do
  for v in 3 2; do
    echo "C5 winv=$v $(KATS_BP_WINV=$v timeout 150 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3))')"
  done
done
KATS_BP_WINV=3 timeout 120 python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/ni4_prof.log 2>&1 && \
KATS_BP_WINV=3 ncu --set full --clock-control none --import-source on -k regex:"^k_bp_window$" -s 0 -c 1 -o gpurun_out/k5c5_ni4 -f python scripts/prof_step.py --config C5 --reps 1 >> gpurun_out/ni4_prof.log 2>&1
