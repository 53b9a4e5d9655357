set -x
python -c "import __graft_entry__ as g; g.build()"
nproc; free -g | head -2; lscpu | grep -i "model name"
BFS_HOST_LOOP=1 timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:k_td_expand|k_bu_batch|k_emit_perm|k_td_finish' -c 14 -o gpurun_out/r02_k29_hub python tools/profile_run.py --config k29 --reindex 1 --root 452924735 --roots 1 > gpurun_out/r02_prof.log 2>&1
echo ncu_rc=$?
tail -5 gpurun_out/r02_prof.log
