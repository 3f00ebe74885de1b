# step-7 kernel choice per config: default vs each kernel forced
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
for cfg in C1 C3; do
  for kk in default window tmem l1; do
    if [ $kk = default ]; then unset KATS_BP_KERNEL; else export KATS_BP_KERNEL=$kk; fi
    echo "$cfg $kk $(timeout 200 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), "K5", round(r["k5_busy_ms_per_step"],4), r["kernel"])')"
  done
  unset KATS_BP_KERNEL
done
