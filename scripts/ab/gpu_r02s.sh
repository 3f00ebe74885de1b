# device entry point: one K5 launch after all filtering vs pipelined per pitch (KATS_PIPELINE=1) or per pitch pair (=2)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_s.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pipelined" > gpurun_out/s_tests.log 2>&1; echo rc=$? >> gpurun_out/s_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3))'; }
for r in 1 2; do for c in C4 C2; do for m in 0 1 2; do echo "$c pipeline=$m $(KATS_PIPELINE=$m b $c)"; done; done; done > gpurun_out/s.log 2>&1
