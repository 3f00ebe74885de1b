# A/B: K4^T over one vs two views per thread (KATS_K4T_VPB); adjoint parity first
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_adjoint.py -m gpu -q > gpurun_out/k4t_test.log 2>&1; echo rc=$? >> gpurun_out/k4t_test.log
for cfg in C5 C2 C3 C5 C2; do
  for v in 1 2; do
    echo "$cfg k4t=$v $(KATS_K4T_VPB=$v timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); a=d["adjoint"]; print(round(a["ms_per_step"],3), round(a["k5T_ms_per_step"],3))')"
  done
done
