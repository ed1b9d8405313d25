"""Dev tool: one case of tests/test_fuzz.py::test_fuzz_batches in a fresh process (so a device
fault cannot poison the next case).  Usage: python tools/fuzz_batch_one.py SEED [N_CASES]
Runs cases SEED..SEED+N-1 with parameters drawn from the seed; prints the first failure."""
import subprocess
import sys

if len(sys.argv) > 2 and sys.argv[2] != "-":
    s0, cnt = int(sys.argv[1]), int(sys.argv[2])
    for s in range(s0, s0 + cnt):
        r = subprocess.run([sys.executable, __file__, str(s), "-"], capture_output=True, text=True)
        if r.returncode != 0:
            print("FAIL", s, r.stdout[-2000:], r.stderr[-1500:])
            sys.exit(1)
    print("all ok")
    sys.exit(0)

import numpy as np  # noqa: E402

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_fuzz as T  # noqa: E402

seed = int(sys.argv[1])
r = np.random.default_rng(seed)
p = dict(nseg=int(r.integers(1, 3000)), long_frac=float(r.choice([0.0, 0.01, 0.2, 1.0])),
         kind=str(r.choice(["classes", "sorted_small", "sorted_wide", "constant", "bytes"])),
         delta=bool(r.integers(0, 2)), seed=int(r.integers(0, 2**31)), gap_in=bool(r.integers(0, 2)),
         gap_out=bool(r.integers(0, 2)), ring=int(r.choice([0, 8, 11, 16])), occ=int(r.choice([0, 1, 3])),
         hint=bool(r.integers(0, 2)))
print(p, flush=True)
import ctypes as C  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402
import torch  # noqa: E402
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
T.test_fuzz_batches.hypothesis.inner_test((torch, lib, DeviceCodec(0)), **p)
print("ok")
