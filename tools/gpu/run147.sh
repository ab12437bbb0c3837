mkdir -p gpurun_out/r147
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r147/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r147/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r147/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r147/bench_default.json 2> gpurun_out/r147/bench_default.err; echo "bench rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r147/bench_torchrun1.json 2> gpurun_out/r147/bench_torchrun1.err; echo "torchrun rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r147/bench_reference.json 2> gpurun_out/r147/bench_reference.err; echo "reference rc=$?"
for pr in bf16 tf32; do timeout 300 python bench.py --prec $pr --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r147/bench_cfg2_$pr.json 2> gpurun_out/r147/bench_cfg2_$pr.err; echo "cfg2 $pr rc=$?"; done
