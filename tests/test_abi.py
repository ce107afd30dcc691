"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol
include/nb.h declares (no compute calls without a GPU), and the header/binding agree."""
import ctypes as C
import os
import re

import paper_2503_02134_b200 as nb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "nb.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(nb_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_abi():
    syms = header_symbols()
    assert set(syms) == set(nb.EXPORTED), syms


def test_library_exports_every_symbol():
    L = C.CDLL(nb._build.build())
    for s in header_symbols():
        assert hasattr(L, s), s
    assert nb.nb_version().startswith("nb-b200")


def test_struct_layouts_match_header():
    # nb_cg_opts / nb_cg_report / nb_info sizes as laid out by a C compiler
    import subprocess, tempfile
    prog = r'''
#include <stdio.h>
#include "nb.h"
int main(void){printf("%zu %zu %zu\n", sizeof(nb_info), sizeof(nb_cg_opts), sizeof(nb_cg_report));return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split()
    assert [int(v) for v in out] == [C.sizeof(nb.nb_info), C.sizeof(nb.nb_cg_opts), C.sizeof(nb.nb_cg_report)]


def test_no_cpu_fallback_without_device():
    """On a machine without a usable GPU the product path fails loudly (never computes on CPU)."""
    h = C.c_void_p()
    rc = nb.lib().nb_setup(2, 2, 2, 3, 0.0, 0, 0, C.byref(h))
    try:
        import torch
        have = torch.cuda.is_available()
    except Exception:
        have = False
    if not have:
        assert rc == nb.NB_ECUDA or rc == nb.NB_EINVAL
        assert nb.nb_last_error()
    else:
        assert rc == nb.NB_OK
        nb.nb_destroy(h)
