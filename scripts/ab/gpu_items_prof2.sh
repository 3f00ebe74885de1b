cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
KATS_BP_ITEMS=4 timeout 120 python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/prof_items.log 2>&1 && \
KATS_BP_ITEMS=4 ncu --set full --clock-control none --import-source on -k regex:"k_bp_items_reg" -s 0 -c 1 \
    -o gpurun_out/k5itemsreg_C5 -f python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/ncu_items.log 2>&1
echo done
