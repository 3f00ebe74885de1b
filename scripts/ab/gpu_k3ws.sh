# A/B: the warp-specialized Hilbert (ws) on narrow detectors (C4, C2, C1) vs the default
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
for cfg in C4 C2 C1; do
  for h in default ws hk; do
    if [ $h = default ]; then unset KATS_HILBERT; else export KATS_HILBERT=$h; fi
    echo "$cfg $h $(KATS_FILTER_STREAMS=1 timeout 300 python scripts/stage_times.py --config $cfg 2>&1 | tail -1)"
    echo "$cfg $h bench $(timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3))')"
  done
done
unset KATS_HILBERT
