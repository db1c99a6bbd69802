# usage: bash scripts/ab_trees.sh tag   (GPU box): per-class cost of the old worktree (_old/) vs
# the current tree, interleaved twice
tag=$1
for rep in 1 2; do
  echo "== old (rep $rep)"; (cd _old && timeout 600 python scripts/trial_cost.py 20000 2>&1 | grep "r=")
  echo "== new (rep $rep)"; timeout 600 python scripts/trial_cost.py 20000 2>&1 | grep "r="
done > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
