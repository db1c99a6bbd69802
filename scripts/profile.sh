# usage: bash scripts/profile.sh tag [queries] [trials]  (on the GPU box; one GPU)
tag=${1:-p}; nq=${2:-5000}; nt=${3:-296}
export PATH=/usr/local/cuda/bin:$PATH
# launch list (cold-cache, serialised): shares, not absolutes
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --ncu --queries $nq --trials $nt > gpurun_out/${tag}_launches.log 2>&1
# full set on the replay kernel
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
  -o gpurun_out/${tag}_prof python bench.py --ncu --queries $nq --trials $nt > gpurun_out/${tag}_prof.log 2>&1
tail -3 gpurun_out/${tag}_prof.log
ls -la gpurun_out/
