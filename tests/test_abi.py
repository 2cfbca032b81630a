"""The C ABI (include/vqb.h): the in-tree libvqb.so loads without a GPU, exports every
declared entry point, and the ctypes mirror matches the C struct layouts."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2503_02236_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vqb.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(vqb_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.lib()
    declared = declared_functions()
    assert set(declared) == set(N.EXPORTS), (declared, N.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.vqb_abi_version() == 2
    nm = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", nm, re.M), name


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(VqbTensor), offsetof(VqbTensor, dims),
         offsetof(VqbTensor, d_codes), offsetof(VqbTensor, d_codebooks), offsetof(VqbTensor, max_code),
         sizeof(VqbLaunch), sizeof(VqbUsage), sizeof(VqbPeerComm), offsetof(VqbPeerComm, slot_elems));
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    T = N.VqbTensor
    want = [ctypes.sizeof(T), T.dims.offset, T.d_codes.offset, T.d_codebooks.offset, T.max_code.offset,
            ctypes.sizeof(N.VqbLaunch), ctypes.sizeof(N.VqbUsage), ctypes.sizeof(N.VqbPeerComm),
            N.VqbPeerComm.slot_elems.offset]
    assert got == want


def test_error_mapping_without_gpu():
    """Validation happens before any CUDA call: descriptor errors map onto the
    reference's exception classes with their messages."""
    from paper_2503_02236_b200.errors import ConfigError, ShapeError
    t = N.VqbTensor()
    t.vector_size, t.log2_entries, t.residuals, t.ndim = 3, 8, 1, 2
    t.dims[0], t.dims[1] = 4, 8
    with pytest.raises(ConfigError, match="vector_size"):
        N.check(N.lib().vqb_dequant(t, None, N.F32, None))
    t.vector_size = 4
    t.dims[1] = 6
    t.n_regions = 1
    with pytest.raises(ShapeError, match="not divisible by vector_size"):
        N.check(N.lib().vqb_dequant(t, None, N.F32, None))
    t.dims[1] = 8
    t.layout = N.LAYOUT_PLAIN
    t.codes_bytes = 2
    t.d_codes = 1
    t.d_codebooks = 1
    with pytest.raises(ShapeError, match="truncated"):
        N.check(N.lib().vqb_dequant(t, None, N.F32, None))
    assert N.lib().vqb_layout_bytes(t, N.LAYOUT_GEMV_IL) < 0  # M=4 not a multiple of 16
