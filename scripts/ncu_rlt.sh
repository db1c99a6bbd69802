# usage: bash scripts/ncu_rlt.sh tag   (GPU box) — full ncu capture of an RLT-only replay launch
tag=${1:-rlt}
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
  -o gpurun_out/${tag} python scripts/ncu_case.py rlt 3000 296 > gpurun_out/${tag}.log 2>&1
tail -2 gpurun_out/${tag}.log
