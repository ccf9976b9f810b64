"""The C-ABI library loads (no GPU needed) and exports every symbol
include/stencil_b200.h declares; the ctypes plan layout matches C."""

import os
import re

from paper_1807_03032_b200.backend import runtime

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "include", "stencil_b200.h")


def test_header_exports_loaded():
    lib = runtime.load_library()
    text = open(HDR).read()
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(sc_[a-z_0-9]+)\(",
                       text, re.M)
    assert set(names) == set(runtime.EXPORTS)
    for n in names:
        assert hasattr(lib, n)
    assert lib.sc_version() >= 100
    assert lib.sc_plan_size() == runtime.C.sizeof(runtime.ScPlan)
