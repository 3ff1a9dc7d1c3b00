"""Host-side checks of the C-ABI library (no GPU needed, no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("di.h", "di_test.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(di_[a-z_0-9]+)\s*\(", txt))
    return names


def test_library_exports_every_declared_symbol():
    from tools import build
    build.build()
    lib = ctypes.CDLL(build.SO)
    syms = declared_symbols()
    assert {"di_graph_upload", "di_solve", "di_residual", "di_history"} <= syms
    for s in sorted(syms):
        assert hasattr(lib, s), s


def test_binding_declares_all_symbols():
    import paper_1204_6255_b200 as di
    assert declared_symbols() == set(di.EXPORTED)


def test_last_error_without_gpu():
    """di_graph_upload must fail loudly (no CPU fallback) on argument errors and without a GPU."""
    import paper_1204_6255_b200 as di
    h = ctypes.c_void_p()
    rc = di._lib.di_graph_upload(None, None, 0, 0, 0, None, None, ctypes.byref(h))
    assert rc == di.DI_EINVAL and h.value is None
    assert b"n_nodes" in di._lib.di_last_error()


def test_no_oracle_in_product():
    """The product package never imports or links the oracle (independence rule)."""
    pkg = os.path.join(ROOT, "paper_1204_6255_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert not re.search(r"\boracle\b\s*(import|\.)|import\s+oracle|di_oracle|libdioracle", txt), f


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of di_stats and di_dist have the C layout of include/di.h (size and
    every field offset), compiled here with gcc."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    import paper_1204_6255_b200 as di
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    checks = []
    for cname, py in (("di_stats", di.Stats), ("di_dist", di.Dist)):
        checks.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            checks.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src = tmp_path / "layout.c"
    src.write_text("#include <stddef.h>\n#include <stdio.h>\n#include \"di.h\"\nint main(void) {\n"
                   + "\n".join(checks) + "\nreturn 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(line.split()[:2]): int(line.split()[2]) for line in out if line.strip()}
    for cname, py in (("di_stats", di.Stats), ("di_dist", di.Dist)):
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
