# C3 step-7 investigation: bench (auto VP), plain run, then one ncu --set full capture of K5 on C3
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
KATS_VERBOSE=1 timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/c3.json 2> gpurun_out/c3.err
timeout 120 python scripts/prof_step.py --config C3 --pitches 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bp_tmem|k_bp_window|k_backproject" -s 1 -c 1 -o gpurun_out/prof_k5_c3 -f python scripts/prof_step.py --config C3 --pitches 1 > gpurun_out/ncu_k5.log 2>&1
echo done
