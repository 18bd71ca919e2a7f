"""Performance-regression guard on the ptxas report of the last in-tree build
(paper_2411_00742_b200/build_pbe.log, written by build.py): the hot kernels must not spill
beyond small, measured-harmless amounts.  A 700-byte spill in k_resident<8,8,256> once cost
30% of the C5 throughput without failing any numerical test."""
import os
import re

import pytest

LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2411_00742_b200",
                   "build_pbe.log")

# mangled kernel -> max spill-store bytes (measured: C5 8 B, fused 2D 24-36 B, temporal blocking 124 B,
# plain streaming 80 B (scalar phase only), adjoint 0 B)
LIMITS = {
    "_ZN3pbe10k_residentILi8ELi8ELi256ELb0ELi1EEEvNS_7KParamsE": 128,    # C5 lockstep (PBE_WS=0): 96 B, same 7.1e10
    "_ZN3pbe13k_resident_wsILi8ELi9ELi256ELb0ELb0ELi0EEEvNS_7KParamsE": 96,   # C5 (bench headline; 74 B: loop scalars)
    "_ZN3pbe10k_2d_fusedENS_9Params2DFE": 96,                             # NEXT-1
    "_ZN3pbe11k_stream_tbENS_14StreamTBParamsE": 256,                     # NEXT-4 (C4 default)
    "_ZN3pbe8k_streamILi0ELb1EEEvNS_12StreamParamsE": 160,                # C4 plain streaming (dynamic tiles)
    "_ZN3pbe9k_adjointILi2ELi64ELb1EEEvNS_9AdjParamsE": 64,              # NEXT-3 (16-CTA clusters)
    "_ZN3pbe9k_adjointILi8ELi256ELb0EEEvNS_9AdjParamsE": 64,             # NEXT-3 single-CTA (PBE_ADJ_CLUSTER=0)
}


def _spills():
    if not os.path.exists(LOG):
        pytest.skip("no build log (build with __graft_entry__.build())")
    txt = open(LOG).read()
    out = {}
    for m in re.finditer(r"Compiling entry function '(\S+)' for 'sm_100a'\n.*?\n\s+(\d+) bytes stack frame, (\d+) bytes "
                         r"spill stores, (\d+) bytes spill loads", txt):
        out[m.group(1)] = int(m.group(3))
    return out


@pytest.mark.parametrize("name", sorted(LIMITS))
def test_hot_kernel_spills_bounded(name):
    sp = _spills()
    assert name in sp, f"{name} not in the build log"
    assert sp[name] <= LIMITS[name], f"{name}: {sp[name]} bytes of spill stores (limit {LIMITS[name]})"
