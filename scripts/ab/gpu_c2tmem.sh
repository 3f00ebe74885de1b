# A/B: C2 with the TMEM kernel (pitch pairs) vs the window kernel (default, W = 32)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
for r in 1 2; do
  for kk in tmem window; do
    echo "C2 $kk $(KATS_BP_KERNEL=$kk timeout 200 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5", round(r["k5_busy_ms_per_step"],3), r["kernel"])')"
  done
done
