# same-box A/B with tools/level_times.py: ab_old/ (git worktree at the previous commit) vs the working tree
# usage: bash tools/ab_levels.sh [ROOTS]
R=${1:-32}
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  (cd ab_old && timeout 900 python tools/level_times.py --roots $R --tag old$i 2>&1 | tail -1 | cut -c1-150)
  timeout 900 python tools/level_times.py --roots $R --tag new$i 2>&1 | tail -1 | cut -c1-150
done
