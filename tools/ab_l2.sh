mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for i in 1 2; do
  for v in 1 0; do
    BFS_L2_PERSIST=$v timeout 700 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --levels-out gpurun_out/levels_k29_p$v.json | cut -c1-90 | sed "s/^/persist=$v /" >> gpurun_out/ab.txt 2>&1
  done
done
python -c "import torch; print('persistingL2CacheMaxSize', torch.cuda.get_device_properties(0).persisting_l2_cache_max_size if hasattr(torch.cuda.get_device_properties(0),'persisting_l2_cache_max_size') else 'n/a')" >> gpurun_out/ab.txt 2>&1
