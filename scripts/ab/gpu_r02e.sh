# Final validation: GPU tests, smoke, the C5 bench line (batch chunk), torchrun N=1 strong and weak
set -x
cd $GRAFT_REPO_ROOT
R=r02e
make -s all > gpurun_out/build_$R.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$R.log
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/bench_${R}_C5.json 2> gpurun_out/bench_${R}_C5.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --no-datagen --no-adjoint > gpurun_out/bench_${R}_torchrun.json 2> gpurun_out/bench_${R}_torchrun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 1 --steps 5 --warmup 3 --scaling weak --no-cpu-baseline --no-datagen --no-adjoint > gpurun_out/bench_${R}_weak.json 2> gpurun_out/bench_${R}_weak.err
echo done
