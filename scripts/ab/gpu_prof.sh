set -x
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
python scripts/prof_step.py --config C4 --pitches 1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_backproject -s 1 -c 1 -o gpurun_out/prof_k5_v1 python scripts/prof_step.py --config C4 --pitches 1 > gpurun_out/ncu_k5.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_for_launches.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo done
