# usage: bash scripts/profile_bench.sh tag   (GPU box, one GPU)
# 1. launch list of the default bench command (serialised, cold-cache: shares, not absolutes)
# 2. one `ncu --set full` capture of the full-size config-2 replay launch (bench.py --ncu)
tag=${1:-r1}
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${tag}_launches.log 2>&1
echo "launch list rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
  -o gpurun_out/${tag}_bench_full python bench.py --ncu > gpurun_out/${tag}_bench_full.log 2>&1
echo "full capture rc=$?"
ncu -i gpurun_out/${tag}_bench_full.ncu-rep --page raw --csv > gpurun_out/${tag}_bench_full_raw.csv 2>&1
tail -2 gpurun_out/${tag}_bench_full.log
