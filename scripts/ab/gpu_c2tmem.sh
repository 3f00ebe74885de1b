cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
for kv in window tmem; do KATS_BP_KERNEL=$kv timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/c2_$kv.json 2>/dev/null; done
KATS_BP_KERNEL=tmem timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "C2 or T2" > gpurun_out/pyt.log 2>&1; echo "rc=$?" >> gpurun_out/pyt.log
echo done
