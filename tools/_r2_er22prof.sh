python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
BFS_HOST_LOOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_bu_batch' -c 2 -o gpurun_out/x_er22 python tools/profile_run.py --config er22 --reindex 1 --roots 1 > gpurun_out/x_er22.log 2>&1; echo rc=$?
