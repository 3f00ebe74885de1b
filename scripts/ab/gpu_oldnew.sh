# same-box A/B of two prebuilt libraries (no rebuild): new, old, new, old on C4
cd $GRAFT_REPO_ROOT
L=paper_2201_02309_b200/libkatsevich.so
cp $L /tmp/new.so
for r in 1 2; do
  cp /tmp/new.so $L; timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/on_new$r.json 2>/dev/null
  cp gpurun_old_libkatsevich.so $L; timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-adjoint --no-datagen > gpurun_out/on_old$r.json 2>/dev/null
done
cp /tmp/new.so $L
echo done
