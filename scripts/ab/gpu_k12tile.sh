# A/B: K12 column walk vs the two-phase shared-memory tile kernel (KATS_K12=tile, tile2, tile4)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "filter_stages or k12" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in ${K12_MODES:-col8 tile}; do for cfg in C4 C3 C5 C2; do
  export KATS_K12=$m
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/k12t_${m}_$cfg.json 2>/dev/null
done; done
if [ -n "$K12_PROF" ]; then
KATS_K12=$K12_PROF timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_deriv_fwd" -s 4 -c 1 \
  -o gpurun_out/k12_$K12_PROF -f python scripts/prof_step.py --config C4 --reps 1 > gpurun_out/ncu_k12_$K12_PROF.log 2>&1
fi
echo done
