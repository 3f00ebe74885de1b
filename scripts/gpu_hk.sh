# warp-specialized Hankel Hilbert: parity, then K3 stage time (ws default vs hk1)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "filter_stages" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in C3 C5 C2; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ws_$cfg.json 2>/dev/null
  KATS_HILBERT=hk1 timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/hk1_$cfg.json 2>/dev/null
done
echo done
