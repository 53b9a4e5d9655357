python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for a in 20 25 30 35 40 50 70; do echo "alpha=$a"; timeout 600 python tools/sweep_env.py --var BFS_NOOP --values 0 --alpha $a 2>&1 | tail -1; done > gpurun_out/al_sweep.txt
cat gpurun_out/al_sweep.txt
