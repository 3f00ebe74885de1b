# compute-sanitizer memcheck over the window kernel's byte ring / row crop, the TMEM kernels and the
# streaming K4^T on small cases (out-of-bounds shared/global accesses would be reported)
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_ab.log 2>&1
export PYTHONFAULTHANDLER=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "window_kernel or pitch_pairs or bp_kernel" > gpurun_out/san1.log 2>&1; echo rc=$? >> gpurun_out/san1.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_flat.py -q -x \
  -k "batch_window or reconstruct_matches or adjoint" > gpurun_out/san2.log 2>&1; echo rc=$? >> gpurun_out/san2.log
