# A/B: adjoint K5^T with the component planes at a compile-time stride (default) vs the runtime stride
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_adjoint.py -q -x > gpurun_out/adjcs_test.log 2>&1; echo "test rc=$?" >> gpurun_out/adjcs_test.log
for cfg in C4 C3 C2; do
  for cs in 1 0; do
    echo "$cfg cs=$cs $(KATS_ADJ_CS=$cs timeout 300 python scripts/adj_perf.py $cfg 2>&1 | tail -1)"
  done
done
for cs in 1 0; do echo "C5 cs=$cs $(KATS_ADJ_CS=$cs timeout 300 python scripts/adj_perf_batch.py C5 2>&1 | tail -1)"; done
