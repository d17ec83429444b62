"""The C-ABI library builds, loads and exports every symbol include/ee.h
declares (no compute calls: runs without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_2312_04916_b200 import _lib, build_lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ee.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ee_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_all_declared_symbols():
    path = build_lib.build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(lib, name), name
    # the ctypes signature table covers exactly the declared ABI
    assert sorted(_lib.SIGNATURES) == syms


def test_abi_metadata_without_gpu():
    lib = _lib.load(build_lib.build())
    assert lib.ee_abi_version() == 1
    # workspace sizing is pure host arithmetic
    assert lib.ee_workspace_bytes(_lib.EE_OP_EXIT_HEAD, 16, 4096, 50304, 32, 2048) > 50304 // 8 * 16 * 12
    # attention: per-chunk partials (4 chunks of 512 positions) + per-(row, head) merge counters
    assert lib.ee_workspace_bytes(_lib.EE_OP_ATTENTION, 8, 4096, 0, 32, 2048) >= 64 * 32 * 4 * 130 * 4
    assert lib.ee_tiled_weight_bytes(4096, 4096) == 4096 * 4096 * 2
    assert lib.ee_tiled_weight_bytes(50304, 4096) == 50304 * 4096 * 2
    assert lib.ee_tiled_weight_bytes(10, 512) == 16 * 512 * 2  # rows padded to 16
    assert lib.ee_tiled_weight_bytes(64, 100) == 0  # not packable


def test_error_codes_map_to_reference_exceptions():
    from paper_2312_04916_b200.errors import ConfigError, NonFiniteError, ShapeError, TokenError
    _lib.load(build_lib.build())
    for rc, exc in ((_lib.EE_ESHAPE, ShapeError), (_lib.EE_ETOKEN, TokenError),
                    (_lib.EE_ENONFINITE, NonFiniteError), (_lib.EE_ECONFIG, ConfigError)):
        with pytest.raises(exc):
            _lib.check(rc, "x")


def test_sm100a_cubin_present():
    """The shared object carries sm_100a SASS (cross-compiled here)."""
    import subprocess
    path = build_lib.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of the ABI structs (`_lib.Ee*`) have the C layout:
    every field offset and the total size, checked against offsetof() from a
    tiny C program compiled against include/ee.h."""
    import subprocess
    structs = {"ee_layer_t": _lib.EeLayer, "ee_decoder_t": _lib.EeDecoder,
               "ee_head_t": _lib.EeHead, "ee_engine_t": _lib.EeEngine,
               "ee_generate_args_t": _lib.EeGenerateArgs}
    lines = ['#include <stdio.h>', '#include <stddef.h>',
             f'#include "{os.path.join(ROOT, "include", "ee.h")}"', 'int main(void) {']
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
