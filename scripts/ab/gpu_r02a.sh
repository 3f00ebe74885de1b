# Round 2, first measurement call: GPU tests, the default bench line (C4), C5 bench, the ncu
# launch list of the bench command, and ncu --set full captures of K12 and K4 (C4, C3, C5).
set -x
cd $GRAFT_REPO_ROOT
R=r02a
make -s all > gpurun_out/build_$R.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$R.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${R}_C5.json 2> gpurun_out/bench_${R}_C5.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/bench_short_$R.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ncu_launches_$R.log 2>&1
for cfg in C4 C3 C5; do
  P=1; [ $cfg = C4 ] && P=8
  timeout 120 python scripts/prof_step.py --config $cfg --pitches $P --reps 1 > gpurun_out/prof_${cfg}_$R.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_deriv_fwd_rebin|k_bwd_rebin_cos" -s 2 -c 2 \
      -o gpurun_out/k12k4_${cfg}_$R -f python scripts/prof_step.py --config $cfg --pitches $P --reps 1 > gpurun_out/ncu_k12k4_${cfg}_$R.log 2>&1
done
echo done
