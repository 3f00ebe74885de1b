# host entry point: tensor-core Hilbert before the first pitch's BP; tests + e2e per config
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host or pipelined" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in C3 C2 C4; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/e2e_$cfg.json 2>/dev/null
done
echo done
