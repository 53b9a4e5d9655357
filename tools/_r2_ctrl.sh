# usage: [CONFIG=k29] bash tools/_r2_ctrl.sh TAG VAR VALUES: sweep on the working tree and on the HEAD export in .ctrl (same box)
TAG=$1; VAR=$2; VALS=$3; CONFIG=${CONFIG:-k29}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
(cd .ctrl && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 && timeout 900 python tools/sweep_env.py --config $CONFIG --var BFS_NOOP --values 0 > ../gpurun_out/${TAG}_ctrl.txt 2>&1)
timeout 900 python tools/sweep_env.py --config $CONFIG --var $VAR --values $VALS > gpurun_out/${TAG}_sweep.txt 2>&1
(cd .ctrl && timeout 900 python tools/sweep_env.py --config $CONFIG --var BFS_NOOP --values 0 >> ../gpurun_out/${TAG}_ctrl.txt 2>&1)
echo "== control (HEAD) $CONFIG"; cat gpurun_out/${TAG}_ctrl.txt; echo "== working tree $CONFIG"; cat gpurun_out/${TAG}_sweep.txt
