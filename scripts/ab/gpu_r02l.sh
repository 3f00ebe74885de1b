# C3: TMEM kernel ring depth (3 CTAs/SM with a 2-slot ring vs 2 CTAs/SM with 4 slots)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_l.log 2>&1 || exit 1
b() { timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants --no-graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["k5_ms_per_launch"],3))'; }
for r in 1 2; do
for kb in 74 110 150; do echo "C3 kb=$kb $(KATS_BP_TMEM_KB=$kb b)"; done
done > gpurun_out/l.log 2>&1
