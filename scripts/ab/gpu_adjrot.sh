# A/B: adjoint K5^T lanes' slice walks rotated by quad row (default) vs by slice; parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_adjoint.py tests/test_gpu_half.py tests/test_gpu_apod.py -q -x > gpurun_out/adjrot_test.log 2>&1; echo "test rc=$?" >> gpurun_out/adjrot_test.log
for cfg in C4 C3 C2; do
  for r in row slice; do
    echo "$cfg rot=$r $(KATS_ADJ_ROT=$r timeout 300 python scripts/adj_perf.py $cfg 2>&1 | tail -1)"
  done
done
for r in row slice; do echo "C5 rot=$r $(KATS_ADJ_ROT=$r timeout 300 python scripts/adj_perf_batch.py C5 2>&1 | tail -1)"; done
timeout 120 python scripts/adj_prof.py C4 > gpurun_out/adjprof3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_bp_adjoint$" -s 0 -c 1 -o gpurun_out/k5T_rot -f python scripts/adj_prof.py C4 >> gpurun_out/adjprof3.log 2>&1
