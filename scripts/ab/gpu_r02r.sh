# C3: two views per pass with a deeper ring at 2 CTAs per SM (KATS_BP_VP=2, KATS_BP_TMEM_KB)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_r.log 2>&1 || exit 1
b() { timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants --no-graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["k5_ms_per_launch"],3))'; }
for r in 1 2; do
echo "C3 default $(b)"
echo "C3 vp2 kb110 $(KATS_BP_VP=2 KATS_BP_TMEM_KB=110 b)"
echo "C3 vp2 kb74 $(KATS_BP_VP=2 b)"
echo "C3 vp2 kb140 $(KATS_BP_VP=2 KATS_BP_TMEM_KB=140 b)"
done > gpurun_out/r.log 2>&1
