# A/B iteration: parity tests on the default BP kernel, bench default vs KATS_BP_KERNEL=window, ncu of the BP kernel
set -x
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
KATS_BP_KERNEL=window timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_alt.json 2> gpurun_out/bench_alt.err
timeout 120 python scripts/prof_step.py --config C4 --pitches 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bp_tmem|k_bp_window|k_backproject" -s 1 -c 1 -o gpurun_out/prof_k5 -f python scripts/prof_step.py --config C4 --pitches 1 > gpurun_out/ncu_k5.log 2>&1
echo done
