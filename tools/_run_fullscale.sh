set -x
python -c "import __graft_entry__ as g; g.build()"
python - <<'PY'
import torch, oracle, paper_1503_04359_b200 as pkg
from tests import fullscale_exact as FX
torch.cuda.set_device(0)
r = FX.serial_oracle_check(pkg, torch, 16, 16, 1, oracle.KRON_ABC, nroots=64)
assert r["depth_equal_all"] and r["validator_failures"] == 0
r = FX.streaming_check(pkg, torch, 18, 16, 1, oracle.KRON_ABC, nroots=16, group=8)
assert r["failures"] == 0
PY
echo smoke_rc=$?
timeout 2000 python tools/fullscale_validate.py --k26-roots 64 --k29-roots 16 --out gpurun_out/r02_fullscale_validation.json
echo full_rc=$?
