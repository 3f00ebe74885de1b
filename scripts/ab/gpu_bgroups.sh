cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "batch" > gpurun_out/bgroups_test.log 2>&1; echo rc=$? >> gpurun_out/bgroups_test.log
for g in 1 2 4 8; do
  for r in 1 2; do
  echo "C5 groups=$g $(KATS_BATCH_GROUPS=$g timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3))')"
  done
done
