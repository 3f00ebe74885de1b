cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
for cfg in C4 C2 C5; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/var_$cfg.json 2> gpurun_out/var_$cfg.err
  echo "$cfg rc=$?"
done
