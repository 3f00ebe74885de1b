set -x
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/bench.json 2> gpurun_out/bench.err
KATS_PIPELINE=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/bench_alt.json 2> gpurun_out/bench_alt.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo done
