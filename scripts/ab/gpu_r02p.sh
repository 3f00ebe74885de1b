# host path (e2e): tensor-core K3 beside the backprojection (KATS_HOST_TC=1) vs the fp32 direct K3
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_p.log 2>&1 || exit 1
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3))'; }
for r in 1 2; do for c in C4 C3 C2; do echo "$c fp32 $(b $c)"; echo "$c tc $(KATS_HOST_TC=1 b $c)"; done; done > gpurun_out/p.log 2>&1
KATS_HOST_TC=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "host" > gpurun_out/p_tests.log 2>&1; echo rc=$? >> gpurun_out/p_tests.log
