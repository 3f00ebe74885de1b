cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 120 python scripts/adj_prof.py C4 > gpurun_out/adjf_prof.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_bwd_rebin_cos_T|k_fwd_rebin_T|k_deriv_T" -s 3 -c 3 -o gpurun_out/adjf -f python scripts/adj_prof.py C4 >> gpurun_out/adjf_prof.log 2>&1
