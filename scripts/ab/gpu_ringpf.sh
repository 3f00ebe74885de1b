# A/B: byte-ring window kernel (C5, four items per CTA) with L2 prefetch of the boxes N views ahead
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
KATS_BP_RING_PF=8 timeout 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -k "c5 or C5 or batch" > gpurun_out/ringpf_test.log 2>&1; echo rc=$? >> gpurun_out/ringpf_test.log
for r in 1 2; do
  for pf in 0 4 8 16; do
    echo "C5 pf=$pf $(KATS_BP_RING_PF=$pf timeout 150 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],3), "K5busy", round(r["k5_busy_ms_per_step"],3), "frac", round(r["frac"],3))')"
  done
done
