"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
entry point include/mk.h declares, and the ctypes mirrors have the C layout."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2604_15379_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mk.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(L.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return L.load()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(mk_\w+)\(", text, re.M)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert "mk_step" in names and "mk_probe" in names and len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(L.EXPORTS) <= set(names)


def test_version_and_error_string_without_gpu(lib):
    assert lib.mk_version() == 1
    assert isinstance(lib.mk_last_error(), bytes)


def test_struct_layouts_match_header(tmp_path):
    structs = {"mk_topology": L.Topology, "mk_task": L.Task, "mk_unit": L.Unit,
               "mk_gemm_params": L.GemmParams, "mk_norm_params": L.NormParams,
               "mk_attn_params": L.AttnParams, "mk_silu_params": L.SiluParams,
               "mk_argmax_params": L.ArgmaxParams, "mk_graph_desc": L.GraphDesc,
               "mk_counters": L.Counters, "mk_log_rec": L.LogRec, "mk_tp_params": L.TPParams}
    src = tmp_path / "sz.c"
    body = "".join(f'printf("{n} %zu\\n", sizeof({n}));' for n in structs)
    src.write_text('#include <stdio.h>\n#include "mk.h"\nint main(void){' + body + "return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    sizes = dict((ln.split()[0], int(ln.split()[1])) for ln in out.strip().splitlines())
    for n, cls in structs.items():
        assert ctypes.sizeof(cls) == sizes[n], n


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
