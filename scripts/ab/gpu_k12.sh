cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "filter_stages or k12" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in rows col8; do for cfg in C4 C3 C5; do
  if [ $m = rows ]; then unset KATS_K12; else export KATS_K12=$m; fi
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/k12_${m}_$cfg.json 2>/dev/null
done; done
echo done
