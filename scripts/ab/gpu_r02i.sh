# C5 slab groups with the batch chunking per group (default 2 groups) vs the device chunk and 1 group
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_i.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flat.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py -m gpu -q -x > gpurun_out/i_tests.log 2>&1; echo rc=$? >> gpurun_out/i_tests.log
b() { timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint --no-variants --no-graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["k5_ms_per_launch"],3))'; }
for r in 1 2; do
echo "default $(b)"
echo "gchunk0 $(KATS_BATCH_GCHUNK=0 b)"
echo "groups1 $(KATS_BATCH_GROUPS=1 b)"
done > gpurun_out/i_groups.log 2>&1
