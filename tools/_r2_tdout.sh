python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 86254516 452924735; do
BFS_HOST_LOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/t_$r.csv python tools/profile_run.py --config k29 --reindex 1 --root $r --roots 1 > gpurun_out/t_$r.log 2>&1; echo rc=$?
done
timeout 600 python tools/td_outlier.py 86254516 452924735 40046910 47537371 515592054 > gpurun_out/t_outlier.txt 2>&1
