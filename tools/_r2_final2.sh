# final round-2 bench + configs + full GPU tests (code after the SWITCH loop graph)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench_rc=$?
for c in k26 er22 k16; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/f_bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --impl reference > gpurun_out/f_ref.json 2>/dev/null; echo ref_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gpu_tests.txt 2>&1; echo pytest_rc=$? >> gpurun_out/f_gpu_tests.txt
tail -2 gpurun_out/f_gpu_tests.txt
