# Round evidence: GPU tests, smoke, bench line, ncu launch list of the bench command, and
# ncu --set full captures of the dominant kernel (as the bench launches it) and of the
# tensor-core Hilbert and the adjoint backprojection.
set -x
cd $GRAFT_REPO_ROOT
R=${ROUND_TAG:-r01}
make -s all > gpurun_out/build.log 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/clocks_$R.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$R.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$R.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ncu_launches_$R.log 2>&1
# full capture: the BP launch of the first timed step (3 warm-up steps -> skip 3 launches)
ncu --set full --clock-control none --import-source on -k regex:"k_bp_tmem|k_bp_window|k_backproject" -s 3 -c 1 \
    -o gpurun_out/k5_full_$R -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ncu_full_$R.log 2>&1
timeout 120 python scripts/stage_times.py --config C4 > gpurun_out/stages_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hilbert_tc2" -s 5 -c 1 \
    -o gpurun_out/k3_full_$R -f python scripts/stage_times.py --config C4 --reps 1 > gpurun_out/ncu_k3_$R.log 2>&1
timeout 120 python scripts/prof_step.py --config C3 > gpurun_out/prof_c3_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hilbert_ws|k_hilbert_hk" -s 2 -c 1 \
    -o gpurun_out/k3hk_full_$R -f python scripts/prof_step.py --config C3 > gpurun_out/ncu_k3hk_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_bp_tmem|k_bp_window" -s 1 -c 1 \
    -o gpurun_out/k5c3_full_$R -f python scripts/prof_step.py --config C3 > gpurun_out/ncu_k5c3_$R.log 2>&1
timeout 120 python scripts/prof_step.py --config C5 > gpurun_out/prof_c5_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bp_tmem|k_bp_window" -s 1 -c 1 \
    -o gpurun_out/k5c5_full_$R -f python scripts/prof_step.py --config C5 > gpurun_out/ncu_k5c5_$R.log 2>&1
timeout 120 python scripts/adj_prof.py C4 > gpurun_out/adjp_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bp_adjoint" -s 2 -c 1 \
    -o gpurun_out/k5T_full_$R -f python scripts/adj_prof.py C4 > gpurun_out/ncu_k5T_$R.log 2>&1
for cfg in C1 C2 C3 C5; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/bench_${R}_$cfg.json 2> gpurun_out/bench_${R}_$cfg.err
done
echo done
