# A/B: K12 warp-per-view vs row form vs round-1 column walk (K4 tile); parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k12 or k4 or batch or reconstruct_matches or filter_stages" > gpurun_out/k12wv_test.log 2>&1; echo rc=$? >> gpurun_out/k12wv_test.log
for cfg in C5 C2 C3 C4; do
  for v in wv rows colv2; do
    echo "$cfg k12=$v $(KATS_K12=$v timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages"]; print(round(d["ms_per_step"],3), "K12", round(f["K12_deriv_fwd_rebin"]["ms_per_step"],3), "K3", round(f["K3_hilbert"]["ms_per_step"],3), "K4", round(f["K4_bwd_rebin_cos"]["ms_per_step"],3))')"
  done
done
