cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
for r in 1 2; do for e in inline pre; do
  KATS_BP_ENDS=$e timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ends_${e}_$r.json 2>/dev/null
done; done
echo done
