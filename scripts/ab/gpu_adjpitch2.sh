cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
for cfg in C4 C3; do
  for m in odd pad32; do
    echo "$cfg $m $(KATS_ADJ_PITCH=$m timeout 300 python scripts/adj_perf.py $cfg 2>&1 | tail -1)"
  done
done
