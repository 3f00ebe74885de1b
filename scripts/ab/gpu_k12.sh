cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
for m in fat col4 col8 col16; do for cfg in C4 C3 C5; do
  KATS_K12=$m timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/k12_${m}_$cfg.json 2>/dev/null
done; done
echo done
