# Round 2 closing measurement call: GPU tests, smoke, bench lines C1-C5 + reference arm, the default
# bench command timed, and the ncu launch list of the C4 and C5 bench commands.
set -x
cd $GRAFT_REPO_ROOT
R=r02zf
make -s all > gpurun_out/build_$R.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$R.log
timeout 900 python bench.py > gpurun_out/bench_default_$R.json 2> gpurun_out/bench_default_$R.err
for cfg in C4 C1 C2 C3 C5; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/bench_${R}_$cfg.json 2> gpurun_out/bench_${R}_$cfg.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen --no-variants --no-graph > gpurun_out/bench_short_$R.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen --no-variants --no-graph > gpurun_out/ncu_launches_$R.log 2>&1
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen --no-variants --no-graph > gpurun_out/bench_short_C5_$R.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5_$R.csv \
    python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen --no-variants --no-graph > gpurun_out/ncu_launches_C5_$R.log 2>&1
echo done
