set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -40 > gpurun_out/t1_tests.log
tail -5 gpurun_out/t1_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/t1_smoke.log 2>&1; tail -3 gpurun_out/t1_smoke.log
timeout 600 python bench.py --queries 20000 --trials 1024 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/t1_bench.log 2>&1; tail -5 gpurun_out/t1_bench.log
