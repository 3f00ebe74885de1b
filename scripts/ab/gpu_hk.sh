# K3 changes: full GPU tests, then K3 stage times and the C5 batch adjoint
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in C3 C5; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-datagen > gpurun_out/ws_$cfg.json 2>/dev/null
done
python scripts/adj_perf_batch.py C5 > gpurun_out/adjb.log 2>&1
echo done
