# A/B: TMEM kernel with pitch pairs (KATS_BP_PP=2) vs single pitches at C4 (and C2 forced TMEM); parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "pitch_pairs or bp_kernel" > gpurun_out/pp_test.log 2>&1; echo rc=$? >> gpurun_out/pp_test.log
KATS_BP_PP=2 timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "c4_all" >> gpurun_out/pp_test.log 2>&1; echo rc=$? >> gpurun_out/pp_test.log
for pp in 2 1 2 1; do
  echo "C4 pp=$pp $(KATS_BP_PP=$pp timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3), "iso", round(r["isolated"]["k5_ms_per_launch"],3))')"
done
for pp in 2 1; do
  echo "C3 pp=$pp (1 pitch: n/a) C2 tmem pp=$pp $(KATS_BP_KERNEL=tmem KATS_BP_PP=$pp timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5busy", round(r["k5_busy_ms_per_step"],3))')"
done
