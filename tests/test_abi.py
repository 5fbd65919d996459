"""The C-ABI library loads on a CPU-only host and exports every entry point
include/ucfvb.h declares; option defaults mirror SolverOptions{}."""
import ctypes as C
import re
from pathlib import Path

from paper_2510_25906_b200 import _abi as A

HEADER = Path(__file__).resolve().parents[1] / "include" / "ucfvb.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ucfvb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_python_mirror_agree():
    assert declared_symbols() == sorted(A.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(A.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version_and_defaults():
    lib = A.load_library()
    assert lib.ucfvb_abi_version() == 1
    o = A.Options()
    lib.ucfvb_options_default(C.byref(o))
    d = A.default_options()
    for f, _ in A.Options._fields_:
        if f == "margins":
            assert tuple(getattr(o.margins, n) for n, _ in A.Margins._fields_) == (1e-4, 0.5, 0.0, 0.0, 5.0, 2.0)
        else:
            assert getattr(o, f) == getattr(d, f), f
    # solver.hpp:29-43 defaults
    assert (o.order, o.mode, o.lambda1p, o.weno_eps, o.weno_b, o.cfl, o.venkat_kappa, o.gamma) == \
        (3, A.HYBRID, 1e3, 1e-3, 4.0, 0.6, 5.0, 1.4)


def test_struct_sizes_match_c_layout():
    # the header's structs are plain C; sizes checked against the ctypes mirror
    assert C.sizeof(A.Options) == 4 * 4 + 6 * 8 + 5 * 8 + 4 + 4 + 8 + 4 + 4
    assert C.sizeof(A.Margins) == 48


HEADER3 = Path(__file__).resolve().parents[1] / "include" / "ucfvb3.h"


def test_3d_library_exports_every_declared_symbol():
    text = re.sub(r"/\*.*?\*/", "", HEADER3.read_text(), flags=re.S)
    syms = sorted(set(re.findall(r"\b(ucfvb3_[a-z0-9_]+)\s*\(", text)))
    assert len(syms) >= 20
    lib = C.CDLL(str(A.LIB_PATH))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2510_25906_b200 import solver3d as S3
    S3.lib()  # every declared 3D symbol has a Python signature
