# usage: bash scripts/profile_c5.sh tag [skip]   (GPU box, one GPU)
# 1. launch list of the default (config-5) bench command: per-launch shares
# 2. one `ncu --set full` capture of the replay launch number `skip` (0 = W=4, 1 = W=8,
#    2 = W=16, 3 = W=32) of the one-step profiling run `bench.py --ncu`
tag=${1:-r2}; skip=${2:-3}
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${tag}_launches.log 2>&1
echo "launch list rc=$?"
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:replay_kernel \
  --launch-skip ${skip} -c 1 -o gpurun_out/${tag}_full python bench.py --ncu > gpurun_out/${tag}_full.log 2>&1
echo "full capture rc=$?"
ncu -i gpurun_out/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_full_raw.csv 2>&1
ncu -i gpurun_out/${tag}_full.ncu-rep --page details --csv > gpurun_out/${tag}_full_details.csv 2>&1
tail -2 gpurun_out/${tag}_full.log
