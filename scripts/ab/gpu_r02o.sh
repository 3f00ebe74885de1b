# K12 row form: views per CTA (KATS_K12R_NVB) at C3 and C4, three CTAs per SM
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_o.log 2>&1 || exit 1
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages_isolated"]["K12_deriv_fwd_rebin"]; print(round(d["ms_per_step"],3), "k12 iso", round(f["ms_per_step"],3), round(f["frac"],3))'; }
for c in C3 C4; do echo "$c default $(b $c)"; for n in 2 4 8 16; do echo "$c nvb=$n $(KATS_K12R_NVB=$n b $c)"; done; done > gpurun_out/o_perf.log 2>&1
