# A/B: K12 row form vs the round-1 column walk, K4 row form vs the round-1 tile kernel; parity first
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "k12 or k4 or batch or reconstruct_matches or filter_stages or c5 or c4" > gpurun_out/k12k4rows_test.log 2>&1; echo rc=$? >> gpurun_out/k12k4rows_test.log
for cfg in C5 C3 C4 C2; do
  for v in ${K12K4_VARIANTS:-"rows rows" "colv2 tile" "rows tile" "colv2 rows"}; do
    set -- $v
    echo "$cfg k12=$1 k4=$2 $(KATS_K12=$1 KATS_K4=$2 timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages"]; print(round(d["ms_per_step"],3), (d.get("e2e") or {}).get("ms_per_step"), "K12", round(f["K12_deriv_fwd_rebin"]["ms_per_step"],3), "K3", round(f["K3_hilbert"]["ms_per_step"],3), "K4", round(f["K4_bwd_rebin_cos"]["ms_per_step"],3))')"
  done
done
