# A/B on one box: ab_old/ (a git worktree at the previous commit) vs the working tree.
# usage: bash tools/ab.sh [extra bench args]
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for i in 1 2 3; do
  (cd ab_old && timeout 700 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" | cut -c1-90 | sed "s/^/old /") >> gpurun_out/ab.txt 2>&1
  timeout 700 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --levels-out gpurun_out/levels_ab.json "$@" | cut -c1-90 | sed "s/^/new /" >> gpurun_out/ab.txt 2>&1
done
