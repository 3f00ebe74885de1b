cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 120 python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/prof_k3c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hilbert_ws" -s 1 -c 1 \
    -o gpurun_out/k3ws_C5 -f python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/ncu_k3ws.log 2>&1
echo done
