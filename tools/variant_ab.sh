# usage: bash tools/variant_ab.sh NAME 'sed-expr' FILE [ENV=VAL ...] -- builds a copy of the repo with the
# sed applied to FILE and prints tools/level_times.py for it (A/B of compile-time knobs on one box)
name=$1; expr=$2; file=$3; shift 3
d=/tmp/variant_$name
rm -rf $d; mkdir -p $d
cp -r $GRAFT_REPO_ROOT/. $d/ 2>/dev/null || cp -r /root/repo/. $d/
cd $d
[ -n "$expr" ] && sed -i "$expr" $file
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "$name build failed"; exit 1; }
env "$@" timeout 900 python tools/level_times.py --roots ${ROOTS:-32} --tag $name
