# C5: uneven slab groups (KATS_BATCH_SPLIT)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_k.log 2>&1 || exit 1
b() { timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants --no-graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3))'; }
for r in 1 2; do
for sp in 8,8 4,12 12,4 4,4,8 4,8,4 8,4,4 4,4,4,4 16; do
echo "split=$sp $(KATS_BATCH_SPLIT=$sp b)"
done
done > gpurun_out/k_split.log 2>&1
