cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 120 python scripts/adj_prof.py C4 > gpurun_out/adjprof2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_bp_adjoint$" -s 0 -c 1 -o gpurun_out/k5T_full_r02 -f python scripts/adj_prof.py C4 >> gpurun_out/adjprof2.log 2>&1
