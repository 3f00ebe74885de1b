# A/B: adjoint K4^T streaming (default where T_br is monotone) vs the read-modify-write kernel
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_adjoint.py tests/test_gpu_half.py tests/test_gpu_apod.py tests/test_gpu_flat.py -q -x > gpurun_out/k4ts_test.log 2>&1; echo rc=$? >> gpurun_out/k4ts_test.log
for cfg in C4 C3; do
  for k in stream rmw; do
    echo "$cfg k4t=$k $(KATS_K4T=$k timeout 300 python scripts/adj_perf.py $cfg 2>&1 | tail -1)"
  done
done
for k in stream rmw; do echo "C5 k4t=$k $(KATS_K4T=$k timeout 300 python scripts/adj_perf_batch.py C5 2>&1 | tail -1)"; done
