# A/B: warp-specialized K3 with three converted A stages (KATS_WS_STAGES=3) vs two; parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
KATS_WS_STAGES=3 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "filter_stages or reconstruct_matches" > gpurun_out/wsst_test.log 2>&1; echo rc=$? >> gpurun_out/wsst_test.log
for r in 1 2; do
  for cfg in C5 C3 C4; do
    for st in 3 2; do
      echo "$cfg stages=$st $(KATS_WS_STAGES=$st timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages_isolated"]; print(round(d["ms_per_step"],3), "K3iso", round(f["K3_hilbert"]["ms_per_step"],3))')"
    done
  done
done
