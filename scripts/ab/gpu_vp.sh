# A/B: view pairs in the TMEM backprojection (automatic choice) vs one view per pass (KATS_BP_VP=1)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in C4 C3 C1 C2; do
  KATS_BP_VP=1 timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/vp1_$cfg.json 2> gpurun_out/vp1_$cfg.err
  KATS_VERBOSE=1 timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/vp2_$cfg.json 2> gpurun_out/vp2_$cfg.err
done
echo done
