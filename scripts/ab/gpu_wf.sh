# window kernel variant sweep (KATS_BP_WINV) on C5 and C2
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "variant or batch" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 2 3; do KATS_BP_WINV=$v timeout 300 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/wv${v}_C5.json 2>/dev/null; done
for v in 0 3; do KATS_BP_WINV=$v timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/wv${v}_C2.json 2>/dev/null; done
echo done
