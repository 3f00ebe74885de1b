# K12 row form: registers / CTAs per SM (KATS_K12R_MINB) at C3 and C4
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_n.log 2>&1 || exit 1
KATS_K12R_MINB=4 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stage or filter or reconstruct" > gpurun_out/n_tests.log 2>&1; echo rc=$? >> gpurun_out/n_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages_isolated"]["K12_deriv_fwd_rebin"]; print(round(d["ms_per_step"],3), "k12 iso", round(f["ms_per_step"],3), round(f["frac"],3))'; }
for r in 1 2; do for c in C3 C4; do for m in 2 3 4; do echo "$c minb=$m $(KATS_K12R_MINB=$m b $c)"; done; done; done > gpurun_out/n_perf.log 2>&1
