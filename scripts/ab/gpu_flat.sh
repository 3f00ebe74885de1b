# Flat-detector variant: GPU parity, then the whole GPU suite and the curved bench lines (the flat
# support adds one multiply per view to the step-7 geometry: C3/C4/C5 must be unchanged)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_flat.py -q -x > gpurun_out/flat_test.log 2>&1; echo rc=$? >> gpurun_out/flat_test.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/flat_all.log 2>&1; echo rc=$? >> gpurun_out/flat_all.log
for cfg in C4 C3 C5; do
  echo "$cfg $(timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3))')"
done
