# usage: bash scripts/ab_c5.sh tag W-list name1 name2 ...   (GPU box): config-5 launches (full
# 16,384-trial lists, tier 1/auto) with each prebuilt library (libkvr.so = "base",
# libkvr_<name>.so otherwise), twice, interleaved
tag=$1; ws=$2; shift 2
for rep in 1 2; do for name in "$@"; do
  lib=paper_2601_18999_b200/libkvr.so; [ "$name" != base ] && lib=paper_2601_18999_b200/libkvr_${name}.so
  echo "== $name (rep $rep)"
  KVR_LIB=$lib KVR_AB_TIERS=0 timeout 900 python scripts/c5_tier_ab.py 1 $ws 2>&1 | grep "M q-r/s"
done; done > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
