cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for o in grid sorted; do for cfg in C3 C2 C5 C4; do
  if [ $o = grid ]; then export KATS_BP_ORDER=grid; else unset KATS_BP_ORDER; fi
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ord_${o}_$cfg.json 2>/dev/null
done; done
echo done
