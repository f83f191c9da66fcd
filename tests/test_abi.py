"""The C-ABI boundary: both shared libraries load without a GPU and export
every entry point include/ispc.h and include/ispc_host.h declare; the ctypes
tables in _native.py cover them all; struct sizes agree between C and
ctypes (checked through the layout-sensitive ABI version and field offsets)."""
import ctypes as C
import os
import re

import pytest

from paper_1904_03383_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DECL = re.compile(r"^[A-Za-z_][\w \*]*?\b(ispc_\w+)\s*\(", re.M)


def declared(header: str) -> set[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return {m.group(1) for m in DECL.finditer(text)}


@pytest.mark.parametrize("header,loader,table", [
    ("ispc.h", N.ispc, N.ISPC_SYMBOLS),
    ("ispc_host.h", N.host, N.HOST_SYMBOLS),
])
def test_every_declared_symbol_is_exported(header, loader, table):
    names = declared(header)
    assert len(names) > 10
    so = loader()  # the product loader (RTLD_GLOBAL, backend first)
    missing = [n for n in sorted(names) if not hasattr(so, n)]
    assert not missing, missing
    unbound = sorted(names - set(table))
    assert not unbound, unbound


STRUCTS = {"ispc_launch": N.Launch, "ispc_tmap": N.TMap, "ispc_tile_config": N.TileConfig,
           "ispc_kernel_spec": N.KernelSpec, "ispc_problem": N.Problem, "ispc_time_opts": N.TimeOpts,
           "ispc_time_result": N.TimeResult, "ispc_search_config": N.SearchConfig,
           "ispc_search_stats": N.SearchStats, "ispc_nest": N.Nest, "ispc_node": N.Node,
           "ispc_space_stats": N.SpaceStats, "ispc_bound_report": N.BoundReport}


def test_struct_layouts_match_the_header(tmp_path):
    """sizeof of every ABI struct, compiled from the header, equals ctypes'."""
    import subprocess
    src = tmp_path / "sz.c"
    body = "".join(f'  printf("%s %zu\\n", "{k}", sizeof({k}));\n' for k in STRUCTS)
    src.write_text('#include <stdio.h>\n#include "ispc_host.h"\nint main(void) {\n' + body + "  return 0;\n}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = dict(zip(out[0::2], map(int, out[1::2])))
    for name, cls in STRUCTS.items():
        assert sizes[name] == C.sizeof(cls), name
    assert N.ABI_VERSION == 2


def test_no_cpu_fallback_when_library_missing(tmp_path, monkeypatch):
    monkeypatch.setattr(N, "LIBISPC_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(N, "_libs", {})
    with pytest.raises(ImportError):
        N.ispc()
