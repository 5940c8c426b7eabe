"""Static checks on the sm_100a objects of the in-tree build (CPU side, via
cuobjdump).  ptxas 12.9 was seen to emit `LDGSTS ... [R + UR + imm],
desc[UR<odd>]` (a cp.async whose shared address carries a uniform-register
part) for one layout of the 3D spreader's record ring; that encoding raises
a warp "illegal instruction" on the B200.  The shipped objects must not
contain it, in any kernel-width instantiation (the GPU tests only run some)."""

import glob
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_no_cp_async_with_uniform_address_part():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    objs = sorted(glob.glob(os.path.join(ROOT, "build", "obj", "esn_inst_*.o")))
    if not os.path.exists(cuobjdump) or not objs:
        pytest.skip("no cuobjdump or no in-tree objects (run __graft_entry__.build())")
    bad = []
    pat = re.compile(r"LDGSTS[^;]*\[R\d+\+UR\d+")
    for o in objs:
        out = subprocess.run([cuobjdump, "-sass", o], capture_output=True, text=True, timeout=300).stdout
        fn = ""
        for line in out.splitlines():
            if "Function :" in line:
                fn = line.split("Function :")[1].strip()
            elif pat.search(line):
                bad.append((os.path.basename(o), fn, line.strip()[:100]))
    assert not bad, bad[:5]
