# K5^T warp-aggregated atomics (KATS_ADJ_AGG=1) vs the rotated per-lane scatter: adjoint parity + timings
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_m.log 2>&1 || exit 1
KATS_ADJ_AGG=1 timeout 900 python -m pytest tests/test_gpu_adjoint.py tests/test_gpu_flat.py tests/test_gpu_fullsize.py -m gpu -q -x -k "adjoint or dot" > gpurun_out/m_tests.log 2>&1; echo rc=$? >> gpurun_out/m_tests.log
b() { timeout 600 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["adjoint"]["ms_per_step"],3), round(d["adjoint"].get("k5T_ms_per_step",0),3))'; }
for c in C5 C2 C3 C4; do
  echo "$c base $(b $c)"
  echo "$c agg  $(KATS_ADJ_AGG=1 b $c)"
done > gpurun_out/m_perf.log 2>&1
