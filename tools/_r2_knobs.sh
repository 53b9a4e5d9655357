python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in k29 k26 er22; do
  echo "== $c BFS_BU_DENSE"; timeout 900 python tools/sweep_env.py --config $c --var BFS_BU_DENSE --values 256,384,640 2>&1 | grep -v build_ms
  echo "== $c BFS_BU_LONG"; timeout 900 python tools/sweep_env.py --config $c --var BFS_BU_LONG --values 32,64,160 2>&1 | grep -v build_ms
  echo "== $c BFS_TILE_MIN"; timeout 900 python tools/sweep_env.py --config $c --var BFS_TILE_MIN --values 4194304,16777216,67108864 2>&1 | grep -v build_ms
done
