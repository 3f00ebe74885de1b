# one ncu --set full capture of the adjoint step-7 kernel on the C5 batch (after a clean plain run)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 120 python scripts/adj_perf_batch.py C5 > gpurun_out/adjb.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bp_adjoint" -s 2 -c 1 -o gpurun_out/prof_adj_c5 -f python scripts/adj_perf_batch.py C5 > gpurun_out/ncu_adj.log 2>&1
echo done
