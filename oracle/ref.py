"""TEST INFRASTRUCTURE ONLY — the same front-end as ``oracle`` bound to the REFERENCE'S OWN
sources (``oracle/_ref/libgsgp_ref.so``: /root/reference/proj's kernels/grid/interp/solvers/gp
.cpp compiled unmodified, where they lie, against the stand-in Eigen/FFTW/json headers of
``oracle/refshim`` — see its README.md for what that does and does not pin).

``oracle.ref.X`` has the signature of ``oracle.X`` for every function and class of the
restatement's front-end, so a test can run the same comparison against either checker.  The
library is built here by ``make -C oracle ref`` when /root/reference is present and travels
to the GPU box prebuilt; ``available()`` says whether it can be used.
"""
from __future__ import annotations

import importlib.util
import os
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(_HERE, "_ref", "libgsgp_ref.so")
REF_SRC = "/root/reference/proj"


def build_ref(force: bool = False) -> str:
    """Compile the reference sources against the stand-ins (needs /root/reference)."""
    if os.path.isdir(REF_SRC):
        cmd = ["make", "-C", _HERE, "ref"] + (["-B"] if force else [])
        subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
    if not os.path.exists(REF_LIB):
        raise FileNotFoundError(f"{REF_LIB} is not built and {REF_SRC} is absent")
    return REF_LIB


def available() -> bool:
    if os.path.exists(REF_LIB):
        return True
    if os.path.isdir(REF_SRC):
        try:
            build_ref()
        except Exception:  # noqa: BLE001
            return False
    return os.path.exists(REF_LIB)


# a second instance of the front-end module, bound to the reference library
_spec = importlib.util.spec_from_file_location("oracle._ref_front_end", os.path.join(_HERE, "__init__.py"))
_mod = importlib.util.module_from_spec(_spec)
sys.modules[_spec.name] = _mod
_spec.loader.exec_module(_mod)
_mod._LIB_PATH = REF_LIB
_mod.build = build_ref
globals().update({k: v for k, v in vars(_mod).items() if not k.startswith("__") and k not in ("build",)})
build = build_ref


def ref_build_info() -> str:
    import ctypes as C

    L = _mod.lib()
    f = L.orc_ref_build
    f.restype = C.c_char_p
    return f().decode()
