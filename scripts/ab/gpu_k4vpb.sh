# A/B: K4 views per CTA (KATS_K4_VPB); parity first
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k4_views or filter_stages or reconstruct_matches or batch" > gpurun_out/k4vpb_test.log 2>&1; echo rc=$? >> gpurun_out/k4vpb_test.log
for cfg in C5 C4 C3 C2; do
  for v in 1 2 4; do
    echo "$cfg vpb=$v $(KATS_K4_VPB=$v timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), (d.get("e2e") or {}).get("ms_per_step"), round(d["filter_stages"]["K4_bwd_rebin_cos"]["ms_per_step"],3))')"
  done
done
