# last refresh on the final code: launch list, BU traffic, bench, other configs, GPU tests, smoke
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --levels-out gpurun_out/g_levels.json > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo bench_rc=$?
for c in k26 er22 k16; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/g_bench_$c.json 2>/dev/null; done
BFS_HOST_LOOP=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-validate > gpurun_out/g_launches.log 2>&1; echo launches_rc=$?
BFS_HOST_LOOP=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:k_bu_batch' --csv --log-file gpurun_out/g_traffic.csv python tools/profile_run.py --config k29 --reindex 1 --roots 8 > gpurun_out/g_traffic.log 2>&1; echo traffic_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g_gpu_tests.txt 2>&1; echo pytest_rc=$? >> gpurun_out/g_gpu_tests.txt
tail -2 gpurun_out/g_gpu_tests.txt
