# window kernel: tests, then C5 (NI auto vs 1) and C2
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
KATS_BP_NI=1 timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ni1_C5.json 2> gpurun_out/ni1_C5.err
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ni2_C5.json 2> gpurun_out/ni2_C5.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ni2_C2.json 2> gpurun_out/ni2_C2.err
echo done
