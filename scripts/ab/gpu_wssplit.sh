cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
for sp in 2 4 5; do for cfg in C5 C3; do
  KATS_HILBERT_WSSPLIT=$sp timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/wss${sp}_$cfg.json 2>/dev/null
done; done
KATS_HILBERT_WSSPLIT=4 KATS_HILBERT=ws timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "filter_stages" > gpurun_out/pyt.log 2>&1; echo "rc=$?" >> gpurun_out/pyt.log
echo done
