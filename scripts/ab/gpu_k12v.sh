# A/B: K12 column walk over 1 / 2 / 4 views per thread (KATS_K12=col8 | colv2 | colv4); parity first
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k12 or batch or reconstruct_matches" > gpurun_out/k12v_test.log 2>&1; echo rc=$? >> gpurun_out/k12v_test.log
for cfg in C5 C4 C3 C2; do
  for v in col8 colv2 colv4; do
    echo "$cfg k12=$v $(KATS_K12=$v timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), (d.get("e2e") or {}).get("ms_per_step"), round(d["filter_stages"]["K12_deriv_fwd_rebin"]["ms_per_step"],3))')"
  done
done
