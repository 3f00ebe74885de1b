# warp-specialized K3: raw TMA chunks in flight (KATS_WS_RAW 4/6/8) at C4, C3, C5
cd $GRAFT_REPO_ROOT
make -s all > gpurun_out/build_w.log 2>&1 || exit 1
KATS_WS_RAW=8 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hilbert_tc.py -m gpu -q -x -k "stage or filter or hilbert" > gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
b() { timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-datagen --no-variants --no-graph --no-adjoint 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d["filter_stages_isolated"]["K3_hilbert"]; print(round(d["ms_per_step"],3), "k3 iso", round(f["ms_per_step"],3))'; }
for r in 1 2; do for c in C4 C3 C5; do for w in 4 6 8; do echo "$c raw=$w $(KATS_WS_RAW=$w b $c)"; done; done; done > gpurun_out/w.log 2>&1
