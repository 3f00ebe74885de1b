cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build.log 2>&1
for kv in default l1; do
  if [ $kv = default ]; then unset KATS_BP_KERNEL; else export KATS_BP_KERNEL=$kv; fi
  python scripts/adj_perf.py C1 > gpurun_out/adjc1_$kv.log 2>&1
  python scripts/adj_perf.py C2 > gpurun_out/adjc2_$kv.log 2>&1
done
echo done
