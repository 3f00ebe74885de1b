# one ncu --set full capture of the Hankel-core Hilbert on C3 (after a clean plain run)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
export KATS_HILBERT_SPLIT=1
timeout 120 python scripts/prof_step.py --config C3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hilbert_hk" -s 1 -c 1 -o gpurun_out/prof_hk_c3 -f python scripts/prof_step.py --config C3 > gpurun_out/ncu_hk.log 2>&1
echo done
