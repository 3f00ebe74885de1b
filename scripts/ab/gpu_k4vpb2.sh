# A/B with 4x device chunks: K4 views per CTA 2 vs 4 on the short-detector configs
cd $GRAFT_REPO_ROOT
for cfg in C5 C2 C5 C2; do
  for v in 2 4; do
    echo "$cfg vpb=$v $(KATS_K4_VPB=$v timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["filter_stages"]["K4_bwd_rebin_cos"]["ms_per_step"],3))')"
  done
done
