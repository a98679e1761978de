#!/bin/bash
# The GPU test-suite and the every-kernel driver against the CHECKED build
# (make checked: shared/DSMEM bounds checks, asserts, barrier jitter) --
# the stand-in for compute-sanitizer, which is closed on the GPU pool.
#   gpurun --timeout 3000 -- 'bash tools/checked_run.sh TAG'
set -u
TAG=${1:-checked}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export ADMM_B200_LIB=$PWD/paper_1204_0556_b200/libadmm_b200_checked.so
timeout 900 python tools/sanitize.py > $OUT/kernels.log 2>&1; echo "kernels exit $? $(grep -c ADMM_CHECKED $OUT/kernels.log) violations"
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1; echo "pytest exit $? $(tail -1 $OUT/pytest.log)"
grep -h ADMM_CHECKED $OUT/*.log | head -5
# negative control: the checks must fire on a deliberate out-of-bounds read
timeout 300 python - > $OUT/probe.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_1204_0556_b200 import _lib
lib = _lib.load()
print("build flags", lib.admm_build_flags())
out = torch.zeros(1, device="cuda")
_lib.check(lib.admm_checked_probe(0, out.data_ptr(), None)); torch.cuda.synchronize()
print("in-bounds probe ok", out.item())
_lib.check(lib.admm_checked_probe(1, out.data_ptr(), None))
try:
    torch.cuda.synchronize()
    print("out-of-bounds probe NOT caught")
except Exception as e:
    print("out-of-bounds probe caught:", str(e).splitlines()[0])
PY
echo "probe: $(grep -E 'caught|ADMM_CHECKED' $OUT/probe.log | head -3 | tr '\n' ' ')"
