cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_adjoint.py -q -x > gpurun_out/pyt.log 2>&1; echo "rc=$?" >> gpurun_out/pyt.log
KATS_ADJ_PITCH=odd timeout 600 python -m pytest tests/test_gpu_adjoint.py -q -x >> gpurun_out/pyt.log 2>&1; echo "rc=$?" >> gpurun_out/pyt.log
for m in odd pad32; do
  KATS_ADJ_PITCH=$m python scripts/adj_perf.py C2 > gpurun_out/adj2_$m.log 2>&1
done
python scripts/adj_perf_batch.py C5 > gpurun_out/adjb.log 2>&1; python scripts/adj_perf.py C4 > gpurun_out/adj4.log 2>&1; python scripts/adj_perf.py C3 > gpurun_out/adj3.log 2>&1
echo done
