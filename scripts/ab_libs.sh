# usage: bash scripts/ab_libs.sh tag name1 name2 ...   (GPU box): trial_cost.py with each prebuilt
# paper_2601_18999_b200/libkvr_<name>.so (KVR_LIB), twice, interleaved
tag=$1; shift
for rep in 1 2; do for name in "$@"; do
  echo "== $name (rep $rep)"
  KVR_LIB=paper_2601_18999_b200/libkvr_${name}.so timeout 600 python scripts/trial_cost.py ${NQ:-20000} 2>&1 | grep "r="
done; done > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
