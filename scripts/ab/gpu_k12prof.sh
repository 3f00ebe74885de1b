cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
timeout 120 python scripts/prof_step.py --config C4 > gpurun_out/k12p.log 2>&1 || exit 1
for m in col8 tile; do
KATS_K12=$m timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_deriv_fwd" -s 4 -c 1 \
  -o gpurun_out/k12_$m -f python scripts/prof_step.py --config C4 --reps 1 > gpurun_out/ncu_k12_$m.log 2>&1
done
for m in; do for cfg in; do
  KATS_K12=$m timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/k12t_${m}_$cfg.json 2>/dev/null
done; done
echo done
