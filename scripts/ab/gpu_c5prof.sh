# one ncu --set full capture of K5 on C5 (after a clean plain run)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
KATS_VERBOSE=1 timeout 120 python scripts/prof_step.py --config C5 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bp_tmem|k_bp_window|k_backproject" -s 1 -c 1 -o gpurun_out/prof_k5_c5 -f python scripts/prof_step.py --config C5 > gpurun_out/ncu_k5.log 2>&1
echo done
