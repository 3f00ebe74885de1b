cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "batch" > gpurun_out/items_test.log 2>&1; echo rc=$? >> gpurun_out/items_test.log
for v in 8 16 4 0; do
  echo "C5 items=$v $(KATS_BP_ITEMS=$v timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages"]; r=d["roofline"]; print(round(d["ms_per_step"],3), r["kernel"], "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3))')"
done
KATS_BP_ITEMS=8 timeout 120 python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/prof_items.log 2>&1 && \
KATS_BP_ITEMS=8 ncu --set full --clock-control none --import-source on -k regex:"k_bp_items" -s 0 -c 1 \
    -o gpurun_out/k5items2_C5 -f python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/ncu_items.log 2>&1
echo done
