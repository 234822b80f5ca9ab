"""The C-ABI boundary without a GPU: libgx loads, exports every function include/graft_exec.h
declares, the ctypes struct layouts match the C compiler's, and errors map onto the reference's
exception hierarchy."""
import ctypes as C
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2312_10636_b200 import _native as N
from paper_2312_10636_b200.errors import FragserveError, InfeasibleError, ValidationError, raise_for_status

HEADER = ROOT / "include" / "graft_exec.h"


def test_library_exports_every_declared_symbol():
    names = re.findall(r"GX_API\s+int\s+(gx_\w+)\s*\(", HEADER.read_text())
    assert len(names) >= 20
    lib = C.CDLL(str(N.LIB_PATH))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert N.lib().gx_abi_version() == N.ABI_VERSION == 3


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "graft_exec.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(gx_tensor), sizeof(gx_op),"
                   " sizeof(gx_serve_stage), sizeof(gx_serve_route), sizeof(gx_serve_client), sizeof(gx_serve_cfg),"
                   " offsetof(gx_op, w_off));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(N.GxTensor), C.sizeof(N.GxOp), C.sizeof(N.GxServeStage), C.sizeof(N.GxServeRoute),
            C.sizeof(N.GxServeClient), C.sizeof(N.GxServeCfg), N.GxOp.w_off.offset]
    assert got == want


def test_status_codes_map_to_reference_errors():
    with pytest.raises(ValidationError):
        raise_for_status(-1, "bad span")
    with pytest.raises(InfeasibleError):
        raise_for_status(-2, "no SMs")
    with pytest.raises(FragserveError):
        raise_for_status(-3, "cuda")
    assert issubclass(ValidationError, ValueError) and issubclass(InfeasibleError, RuntimeError)


def test_abi_rejects_bad_arguments_without_a_device():
    lib = N.lib()
    h = C.c_void_p()
    cfg = N.GxServeCfg()
    cfg.clock = N.GX_CLOCK_VIRTUAL
    stage = (N.GxServeStage * 1)()
    stage[0].batch, stage[0].instances = 0, 1  # invalid batch
    rc = lib.gx_serve_create(C.c_void_p(1), 1, stage, 0, None, 0, None, C.byref(cfg), C.byref(h))
    assert rc == -1
    assert "batch" in N.last_error()
    with pytest.raises(ValidationError):
        N.check(rc)
