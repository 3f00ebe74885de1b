# host-path tensor-core K3 default: GPU suite + e2e per config
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_q.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3))'; }
for c in C5 C1; do echo "$c tc $(b $c)"; echo "$c fp32 $(KATS_HOST_TC=0 b $c)"; done > gpurun_out/q.log 2>&1
