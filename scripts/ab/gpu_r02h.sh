# C5: slab-group overlap re-measured on the current kernels; ncu of the default window kernel
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_h.log 2>&1 || exit 1
b() { timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants --no-graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["k5_ms_per_launch"],3))'; }
for g in 1 2 4; do for r in 1 2; do echo "C5 groups=$g $(KATS_BATCH_GROUPS=$g b)"; done; done > gpurun_out/h_groups.log 2>&1
timeout 300 python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/h_prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bp_window -c 1 -o gpurun_out/h_k5_c5 -f python scripts/prof_step.py --config C5 --reps 1 > gpurun_out/h_ncu.log 2>&1
echo done
