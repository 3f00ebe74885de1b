# K12 warp-per-view form: g2 row-loop unroll (KATS_K12WV_UR) and views per warp (KATS_K12WV_VPW) at C5 and C2
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_t.log 2>&1 || exit 1
KATS_K12WV_UR=16 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stage or filter or batch" > gpurun_out/t_tests.log 2>&1; echo rc=$? >> gpurun_out/t_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages_isolated"]["K12_deriv_fwd_rebin"]; print(round(d["ms_per_step"],3), "k12 iso", round(f["ms_per_step"],3), round(f["frac"],3))'; }
for r in 1 2; do for c in C5 C2; do
  echo "$c ur4 $(b $c)"; echo "$c ur8 $(KATS_K12WV_UR=8 b $c)"; echo "$c ur16 $(KATS_K12WV_UR=16 b $c)"
  for v in 1 2 4; do echo "$c ur16 vpw$v $(KATS_K12WV_UR=16 KATS_K12WV_VPW=$v b $c)"; done
done; done > gpurun_out/t.log 2>&1
