"""Build-quality checks on the sm_100a machine code of the operator kernels (CPU only:
cuobjdump of the in-tree libtomo.so). A plane step of the operator kernels (from the TMA
mbarrier wait to the plane barrier) must not touch local memory: with the shared-memory
carve-out at its maximum, L1 is small and a spill goes to L2 - measured on the B200, five
spilled loads and two stores per step made the fused PCG launch 89 us instead of 70 us
(DESIGN.md §5.3). The step must also still be what DESIGN.md describes: TMA loads
(UTMALDG), the mbarrier wait, FP64 arithmetic, warp shuffles, no tensor-core instructions."""
import re
import shutil
import subprocess

import pytest

from paper_2104_12282_b200 import build as tbuild

INS = re.compile(r"/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)")


def _functions():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    lib = tbuild.build()
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    out = {}
    for part in re.split(r"\n\s+Function : ", sass)[1:]:
        name = part.split("\n", 1)[0].strip()
        out[name] = [m.group(1) for m in INS.finditer(part)]  # opcodes with modifiers
    return out


@pytest.fixture(scope="module")
def funcs():
    return _functions()


def _kernel(funcs, tag):
    hits = [v for k, v in funcs.items() if tag in k]
    assert len(hits) == 1, (tag, [k for k in funcs if tag in k])
    return hits[0]


def _base(op):
    return op.split(".")[0]


def _steps(ops):
    """Compute parts of the plane steps: from an mbarrier phase wait (the TMA data of a
    plane) to the next block barrier, if it holds the element arithmetic (>= 100 FP64
    instructions; the short waits that drain a pipeline are not steps)."""
    steps = []
    for i, op in enumerate(ops):
        if op.startswith("SYNCS.PHASECHK"):
            j = next((j for j in range(i + 1, min(len(ops), i + 900)) if ops[j].startswith("BAR.SYNC")), None)
            if j is None:
                continue
            s = [_base(o) for o in ops[i:j]]
            if s.count("DADD") + s.count("DFMA") + s.count("DMUL") >= 100:
                steps.append(s)
    return steps


@pytest.mark.parametrize("tag,name", [("k_opILi1E", "fused PCG (k_op<OP_PCG>)"),
                                      ("k_opILi0E", "K_hat u (k_op<OP_APPLY>)")])
def test_operator_plane_steps_do_not_spill(funcs, tag, name):
    ops = _kernel(funcs, tag)
    steps = _steps(ops)
    assert steps, f"{name}: no plane step found"
    for s in steps:
        assert "LDL" not in s and "STL" not in s, f"{name}: local-memory spill in a plane step"
        assert "SHFL" in s and "LDS" in s


@pytest.mark.parametrize("tag", ["k_opILi1E", "k_opILi0E"])
def test_operator_uses_tma_and_no_tensor_cores(funcs, tag):
    ops = [_base(o) for o in _kernel(funcs, tag)]
    assert "UTMALDG" in ops  # cp.async.bulk.tensor (TMA) loads
    assert not any(op.startswith(("HMMA", "DMMA", "UTCMMA", "UTCHMMA", "UTCQMMA")) for op in ops)
