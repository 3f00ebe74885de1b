# A/B: filter chunk size (KATS_FILTER_CHUNK_MUL x the default 256*max(1,128/n_psi) views)
cd $GRAFT_REPO_ROOT
for cfg in C5 C2 C3 C4; do
  for m in 1 2 4; do
    echo "$cfg mul=$m $(KATS_FILTER_CHUNK_MUL=$m timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), (d.get("e2e") or {}).get("ms_per_step"))')"
  done
done
