cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
KATS_BP_SLOTS=3 KATS_BP_KERNEL=tmem timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "variant" >> gpurun_out/pytest_gpu.log 2>&1; echo "pytest3 rc=$?" >> gpurun_out/pytest_gpu.log
KATS_VERBOSE=1 timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/sl_C4.json 2>gpurun_out/sl_C4.err
KATS_BP_SLOTS=4 timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/sl4_C4.json 2>/dev/null
timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/sl_C3.json 2>/dev/null
KATS_BP_SLOTS=3 timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/sl3_C3.json 2>/dev/null
echo done
