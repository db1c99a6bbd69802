# usage: bash scripts/ncu_lru.sh tag   (GPU box) — full ncu capture of a Leaf-LRU-only replay launch
tag=${1:-lru}
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
  -o gpurun_out/${tag} python scripts/ncu_case.py lru 3000 296 > gpurun_out/${tag}.log 2>&1
tail -1 gpurun_out/${tag}.log
