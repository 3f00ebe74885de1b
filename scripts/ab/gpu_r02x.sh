# pitch-pair TMEM kernel with the 4x4 half-warp lane map (KATS_BP_PP_Q44=1, template, no runtime branch): parity + C4/C2
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_x.log 2>&1 || exit 1
KATS_BP_PP_Q44=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/x_tests.log 2>&1; echo rc=$? >> gpurun_out/x_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["k5_ms_per_launch"],3))'; }
for r in 1 2; do for c in C4 C2; do echo "$c rows $(b $c)"; echo "$c q44 $(KATS_BP_PP_Q44=1 b $c)"; done; done > gpurun_out/x.log 2>&1
