# Round evidence: GPU tests, bench line, ncu launch list of the bench command, and one
# ncu --set full capture of the dominant kernel launched exactly as the bench launches it.
set -x
cd $GRAFT_REPO_ROOT
R=${ROUND_TAG:-r01}
make -s all > gpurun_out/build.log 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/clocks_$R.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$R.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_$R.log 2>&1
# full capture: the BP launch of the first timed step (3 warm-up steps -> skip 3 launches)
ncu --set full --clock-control none --import-source on -k regex:"k_bp_tmem|k_bp_window|k_backproject" -s 3 -c 1 \
    -o gpurun_out/k5_full_$R -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$R.log 2>&1
echo done
