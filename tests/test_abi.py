"""CPU checks of the C-ABI boundary: the built library loads, exports every
entry point include/miniba.h declares, and the ctypes struct layouts match
the C compiler's (no device calls)."""
import ctypes as ct
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "miniba.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mba_\w+)\s*\(", src)))


def _lib_path():
    from paper_2506_05558_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2506_05558_b200.build import build
        build()
    return _lib.LIB_PATH


def test_library_exports_every_declared_symbol():
    lib = ct.CDLL(_lib_path())
    declared = _declared()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    from paper_2506_05558_b200 import _lib
    assert set(_lib.EXPORTED) == set(declared)


def test_binding_loads_and_reports_abi_version():
    from paper_2506_05558_b200 import _lib
    _lib_path()
    L = _lib.lib()
    assert L.mba_abi_version() == 1


def test_struct_layouts_match_c(tmp_path):
    from paper_2506_05558_b200._lib import MbaBatchDesc, MbaLmConfig, MbaOutputs
    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "miniba.h"\n'
                 'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(MbaBatchDesc), '
                 'sizeof(MbaLmConfig), sizeof(MbaOutputs), sizeof(MbaObs), '
                 'offsetof(MbaLmConfig, fail_iters_mask), offsetof(MbaBatchDesc, flags));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(c), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ct.sizeof(MbaBatchDesc), ct.sizeof(MbaLmConfig), ct.sizeof(MbaOutputs), 16,
                   MbaLmConfig.fail_iters_mask.offset, MbaBatchDesc.flags.offset]


def test_no_cuda_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import numpy as np
    from gsrecon import miniba as M
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        M.huber_cost(np.ones(4), 2.0)
    p = M.BaProblem(R=np.eye(3)[None], t=np.zeros((1, 3)), focal=500.0, cx=0.0, cy=0.0,
                    points=np.ones((1, 3)), cam_idx=np.zeros(1, int), pt_idx=np.zeros(1, int),
                    uv=np.zeros((1, 2)), fixed_cams=np.array([False]))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        M.lm_solve(p, M.LmConfig())
    with pytest.raises(ValueError):
        M.lm_solve(M.BaProblem(R=np.eye(3)[None], t=np.zeros((1, 3)), focal=1.0, cx=0.0, cy=0.0,
                               points=np.zeros((0, 3)), cam_idx=np.zeros(0, int),
                               pt_idx=np.zeros(0, int), uv=np.zeros((0, 2)),
                               fixed_cams=np.array([True])), M.LmConfig())
