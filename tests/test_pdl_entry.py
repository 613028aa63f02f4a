"""Every CUDA kernel opens with TT_PDL_ENTRY() (griddepcontrol.wait).

Programmatic dependent launch is on by default for eager launches
(engine.cu, pdl_enabled): a kernel may be scheduled while its predecessor
drains, so it must wait before reading the predecessor's output.  The one
kernel that lacked the wait (k_tc_fwd, earlier in round 1) read the plan
before it was complete.  This scans the sources so a new kernel cannot
repeat that.
"""
import os
import re

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2206_10581_b200", "csrc")


def kernels():
    """(file, kernel name, first statements of the body) for every __global__ definition."""
    out = []
    for fn in sorted(os.listdir(CSRC)):
        if not fn.endswith((".cu", ".cuh")):
            continue
        src = open(os.path.join(CSRC, fn)).read()
        for m in re.finditer(r"__global__[^;{]*?\b(k_\w+)\s*\(", src):
            # skip to the opening brace of the body (the parameter list may hold parentheses)
            depth, i = 0, m.end() - 1
            while i < len(src):
                if src[i] == "(":
                    depth += 1
                elif src[i] == ")":
                    depth -= 1
                    if depth == 0:
                        break
                i += 1
            brace = src.find("{", i)
            semi = src.find(";", i)
            if brace < 0 or (0 <= semi < brace):
                continue  # a declaration, not a definition
            body = src[brace + 1: brace + 1 + 600]
            first = [s.strip() for s in body.split(";")[:4]]
            out.append((fn, m.group(1), first))
    return out


def test_kernels_found():
    names = {k for _, k, _ in kernels()}
    for expected in ("k_fused_fwd", "k_fused_bwd", "k_tc_fwd", "k_tc_bwd", "k_scan_onepass", "k_last_level"):
        assert expected in names


def test_every_kernel_waits_for_its_predecessor():
    missing = []
    for fn, name, first in kernels():
        # the wait must come before any statement that could read global memory:
        # allow it among the first few statements (static_asserts / constexprs may precede it)
        if not any("TT_PDL_ENTRY()" in s for s in first):
            missing.append(f"{fn}:{name}")
    assert not missing, "kernels without TT_PDL_ENTRY() at the top: " + ", ".join(missing)
