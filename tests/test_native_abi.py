"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import glob
import os
import re

from conftest import ROOT
from paper_2205_13603_b200 import native


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names |= set(re.findall(r"\b(ls_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("ls_runner_create", "ls_runner_set_workload", "ls_runner_measure",
                 "ls_score_batch", "ls_featurize_batch", "ls_sim_latency_batch",
                 "ls_runner_destroy", "ls_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = native.lib()
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(native.EXPORTS) == declared_symbols()


def test_version_and_error_without_gpu():
    lib = native.lib()
    assert b"sm_100a" in lib.ls_version()
    h = ctypes.c_void_p()
    st = lib.ls_runner_create(0, None, ctypes.byref(h))
    import torch
    if not torch.cuda.is_available():
        assert st == 3  # LS_ERR_CUDA: no CPU fallback
        assert b"no CPU fallback" in lib.ls_last_error()
