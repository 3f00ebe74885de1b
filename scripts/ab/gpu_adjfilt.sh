# A/B: adjoint filter transposes over 4x chunks on two streams (default) vs one stream, base chunk
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/adjfilt_test.log 2>&1; echo rc=$? >> gpurun_out/adjfilt_test.log
for cfg in C5 C2 C3 C4; do
  for mode in new old; do
    if [ $mode = old ]; then export KATS_FILTER_CHUNK_MUL=1 KATS_FILTER_STREAMS=1; else unset KATS_FILTER_CHUNK_MUL KATS_FILTER_STREAMS; fi
    echo "$cfg $mode $(timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-datagen 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); a=d["adjoint"]; print(round(d["ms_per_step"],3), round(a["ms_per_step"],3), round(a["k5T_ms_per_step"],3))')"
  done
  unset KATS_FILTER_CHUNK_MUL KATS_FILTER_STREAMS
done
