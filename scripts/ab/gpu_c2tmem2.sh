# C2 default (now the pitch-pair TMEM kernel) + parity; C5 with the TMEM kernel forced for reference
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c2t_test.log 2>&1; echo rc=$? >> gpurun_out/c2t_test.log
for r in 1 2; do
  echo "C2 default $(timeout 200 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5", round(r["k5_busy_ms_per_step"],3), r["kernel"], "e2e", round(d["e2e"]["ms_per_step"],3))')"
  echo "C5 tmem $(KATS_BP_KERNEL=tmem timeout 200 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5", round(r["k5_busy_ms_per_step"],3), r["kernel"])')"
done
