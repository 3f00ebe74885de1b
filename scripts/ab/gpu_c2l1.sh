cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
for kv in window l1; do KATS_BP_KERNEL=$kv timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/c2_$kv.json 2>/dev/null; done
echo done
