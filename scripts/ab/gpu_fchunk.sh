# A/B: filter chunk size on the device entry points (KATS_FILTER_CHUNK_MUL x the base
# 256*max(1,128/n_psi) views; the host-staged path keeps the base chunk); parity at x4 first
cd $GRAFT_REPO_ROOT
KATS_FILTER_CHUNK_MUL=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/fchunk_test.log 2>&1; echo rc=$? >> gpurun_out/fchunk_test.log
for cfg in C5 C4 C3 C2; do
  for m in 1 2 4 1 2 4; do
    echo "$cfg mul=$m $(KATS_FILTER_CHUNK_MUL=$m timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), (d.get("e2e") or {}).get("ms_per_step"))')"
  done
done
