# A/B after the 4x device filter chunks: Hilbert variant (KATS_HILBERT) on C5 / C3 / C2
cd $GRAFT_REPO_ROOT
for cfg in C5 C3 C2; do
  for h in default ws hk tc default; do
    if [ $h = default ]; then unset KATS_HILBERT; else export KATS_HILBERT=$h; fi
    echo "$cfg hilbert=$h $(timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["filter_stages"]["K3_hilbert"]["ms_per_step"],3))')"
  done
  unset KATS_HILBERT
done
