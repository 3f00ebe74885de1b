# C5: slab groups x window-kernel variant (V=3: four slabs per CTA; V=2: two)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_j.log 2>&1 || exit 1
b() { timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants --no-graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["k5_ms_per_launch"],3))'; }
for r in 1 2; do
for g in 1 2; do
echo "groups=$g V=3 $(KATS_BATCH_GROUPS=$g b)"
echo "groups=$g V=2 $(KATS_BATCH_GROUPS=$g KATS_BP_WINV=2 b)"
done
done > gpurun_out/j.log 2>&1
