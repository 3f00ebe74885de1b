set -x
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/memcheck_small.py > gpurun_out/memcheck_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/memcheck_small.py > gpurun_out/memcheck.log 2>&1
echo done
