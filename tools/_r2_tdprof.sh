python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
BFS_HOST_LOOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_td_expand|k_td_finish|k_tile_rec' --launch-skip 2 -c 4 -o gpurun_out/u_td python tools/profile_run.py --config k29 --reindex 1 --root 452924735 --roots 1 > gpurun_out/u_td.log 2>&1; echo rc=$?
