# K5 TMEM kernel with predicated gathers in masked groups: parity, then C4/C3/C2 step times
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "bp_kernel or c4 or c3 or end_views" > gpurun_out/k5mask_test.log 2>&1; echo rc=$? >> gpurun_out/k5mask_test.log
for cfg in C4 C3; do
  for r in 1 2; do
  echo "$cfg $(timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), r["kernel"], "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3), "iso", round(r["isolated"]["k5_ms_per_launch"],3))')"
  done
done
