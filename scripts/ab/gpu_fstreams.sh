# A/B: filter chunks on one stream (KATS_FILTER_STREAMS=1) vs alternating over two streams (default),
# with the K12 column walk and the tile kernel
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for fs in ${FS_MODES:-1 2}; do for m in ${K12_MODES:-col8}; do for cfg in C4 C3 C5 C2; do
  KATS_FILTER_STREAMS=$fs KATS_K12=$m timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/fs${fs}_${m}_$cfg.json 2>/dev/null
done; done; done
echo done
