# Round 2 measurement call: GPU tests, shared-memory peak microbenchmark, bench lines C1-C5,
# ncu launch list of the bench command, ncu --set full of K12 (round-2 forms) and K5 at C4.
set -x
cd $GRAFT_REPO_ROOT
R=r02b
make -s all > gpurun_out/build_$R.log 2>&1
(cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_peak smem_peak.cu && ./smem_peak && ./smem_peak) > gpurun_out/smem_peak_$R.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$R.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_$R.csv &
CLK=$!
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
for cfg in C1 C2 C3 C5; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/bench_${R}_$cfg.json 2> gpurun_out/bench_${R}_$cfg.err
done
kill $CLK
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err
KATS_FILTER_STREAMS=1 timeout 300 python scripts/stage_times.py --config C4 > gpurun_out/stages_C4_$R.log 2>&1
KATS_FILTER_STREAMS=1 timeout 300 python scripts/stage_times.py --config C3 > gpurun_out/stages_C3_$R.log 2>&1
KATS_FILTER_STREAMS=1 timeout 300 python scripts/stage_times.py --config C5 > gpurun_out/stages_C5_$R.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/bench_short_$R.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/ncu_launches_$R.log 2>&1
for cfg in C4 C3 C5; do
  P=1; [ $cfg = C4 ] && P=8
  timeout 120 python scripts/prof_step.py --config $cfg --pitches $P --reps 1 > gpurun_out/prof_${cfg}_$R.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_deriv_fwd_rebin" -s 1 -c 1 \
      -o gpurun_out/k12_${cfg}_$R -f python scripts/prof_step.py --config $cfg --pitches $P --reps 1 > gpurun_out/ncu_k12_${cfg}_$R.log 2>&1
done
echo done
