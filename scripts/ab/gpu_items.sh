# C5 items kernel: parity first, then A/B against the register-window kernel (V=2)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "batch or c5" > gpurun_out/items_test.log 2>&1; echo rc=$? >> gpurun_out/items_test.log
for v in 8 4 16 2 0; do
  echo "C5 items=$v $(KATS_BP_ITEMS=$v timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages"]; r=d["roofline"]; print(round(d["ms_per_step"],3), r["kernel"], "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3), "adj", round(d["adjoint"]["ms_per_step"],3))')"
done
