# A/B: batch filter chunk = half the batch's views (default) vs the device chunk (KATS_BATCH_CHUNK=0); parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "batch or c5 or C5" > gpurun_out/bchunk_test.log 2>&1; echo rc=$? >> gpurun_out/bchunk_test.log
for r in 1 2; do
  for b in 1 0; do
    echo "C5 batch_chunk=$b $(KATS_BATCH_CHUNK=$b timeout 200 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3))')"
  done
done
