# one ncu --set full capture of the warp-specialized Hilbert on C5 (after a clean plain run)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 120 python scripts/prof_step.py --config C5 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hilbert_ws" -s 1 -c 1 -o gpurun_out/prof_ws_c5 -f python scripts/prof_step.py --config C5 > gpurun_out/ncu_ws.log 2>&1
echo done
