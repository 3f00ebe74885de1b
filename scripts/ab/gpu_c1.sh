cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for cfg in C1 C2; do
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/c1_$cfg.json 2>/dev/null
done
echo done
