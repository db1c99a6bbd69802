# usage: bash scripts/ab_variants.sh tag "name1:DEF1,DEF2" "name2:" ...   (GPU box)
# builds each variant and runs scripts/trial_cost.py with it
tag=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  lib=$(python -c "
import sys; sys.path.insert(0, '.')
from paper_2601_18999_b200 import build
print(build.build_variant('$name', [d for d in '$defs'.split(',') if d]))")
  echo "== $name ($defs)"
  KVR_LIB=$lib timeout 600 python scripts/trial_cost.py ${NQ:-20000} 2>&1 | grep "r="
done > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
