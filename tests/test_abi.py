"""The C-ABI library loads without a GPU and exports every symbol the public
header declares; the ctypes mirror of the structs matches the header."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "taser_b200.h")
LIB = os.path.join(ROOT, "paper_2402_05396_b200", "libtaser_b200.so")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|unsigned long long)\s+(tg_\w+)\s*\(", text, re.M)))


def test_header_declares_the_path():
    names = declared_functions()
    for required in ("tg_tcsr_build", "tg_find", "tg_lookup_gather", "tg_cache_replace", "tg_sample_wor"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    from paper_2402_05396_b200 import _lib
    assert set(declared_functions()) == set(_lib._SIGNATURES)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_abi_version_and_error_plumbing():
    from paper_2402_05396_b200 import _lib
    assert _lib.lib.tg_abi_version() == _lib.ABI_VERSION == 4
    a = _lib.tg_find_args()
    a.m = 0
    rc = _lib.lib.tg_find(_lib.tg_graph(), a, None, None, None)
    assert rc == _lib.TG_EVALUE
    assert b"budget" in _lib.lib.tg_last_error()


def test_struct_layout_matches_header():
    """Compile a tiny C program against the header that prints sizeof/offsetof
    and compare with the ctypes Structures."""
    from paper_2402_05396_b200 import _lib
    src = r'''
    #include <stdio.h>
    #include <stddef.h>
    #include "taser_b200.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu %zu\n", sizeof(tg_rowmap), sizeof(tg_graph), sizeof(tg_feat_store),
             sizeof(tg_cache_dev), sizeof(tg_find_args), sizeof(tg_pcg64));
      printf("%zu %zu %zu\n", offsetof(tg_find_args, rows), offsetof(tg_find_args, feat_ld),
             offsetof(tg_find_args, window));
      return 0;
    }'''
    tmp = "/tmp/tg_layout"
    with open(tmp + ".c", "w") as fh:
        fh.write(src)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), tmp + ".c", "-o", tmp], check=True)
    out = subprocess.run([tmp], capture_output=True, text=True).stdout.split()
    sizes = [ctypes.sizeof(s) for s in (_lib.tg_rowmap, _lib.tg_graph, _lib.tg_feat_store, _lib.tg_cache_dev,
                                         _lib.tg_find_args, _lib.tg_pcg64)]
    offs = [_lib.tg_find_args.rows.offset, _lib.tg_find_args.feat_ld.offset, _lib.tg_find_args.window.offset]
    assert [int(x) for x in out] == sizes + offs
