cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
KATS_BP_ITEMS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "batch_items or batch_matches" > gpurun_out/items3_test.log 2>&1; echo rc=$? >> gpurun_out/items3_test.log
for v in 4 0 4 0; do
  echo "C5 items=$v $(KATS_BP_ITEMS=$v timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), r["kernel"], "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3))')"
done
