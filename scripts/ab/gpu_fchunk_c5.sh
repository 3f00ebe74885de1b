# A/B: filter chunk size at C5 (KATS_FILTER_CHUNK_MUL x 768 views): L2 residency of g3/g4 vs fuller launches
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
for r in 1 2; do
  for m in 1 2 4 8 12; do
    echo "C5 mul=$m $(KATS_FILTER_CHUNK_MUL=$m timeout 200 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages"]; print(round(d["ms_per_step"],3), "K5", round(d["roofline"]["k5_busy_ms_per_step"],3), "K12", round(f["K12_deriv_fwd_rebin"]["ms_per_step"],3), "K3", round(f["K3_hilbert"]["ms_per_step"],3), "K4", round(f["K4_bwd_rebin_cos"]["ms_per_step"],3))')"
  done
done
