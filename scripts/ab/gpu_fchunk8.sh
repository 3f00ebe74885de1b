# A/B: device filter chunk x4 (default) vs x8 / x2
cd $GRAFT_REPO_ROOT
for cfg in C5 C3 C2 C4 C5 C3; do
  for m in 4 8; do
    echo "$cfg mul=$m $(KATS_FILTER_CHUNK_MUL=$m timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3))')"
  done
done
