"""C-ABI checks that need no GPU: the library loads, exports every symbol include/girg.h
declares, validates arguments before any launch, and the product path is independent of the
oracle (no import, no link, no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "girg.h")


@pytest.fixture(scope="module")
def girg():
    import __graft_entry__

    __graft_entry__._builder().build()
    import paper_1905_06706_b200 as g

    return g


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(girg_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("girg_weights", "girg_positions", "girg_scale_weights", "girg_edges", "girg_strerror"):
        assert f in names


def test_library_exports_every_declared_symbol(girg):
    lib = C.CDLL(girg.library_path())
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", girg.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (girg_\w+)", out))
    assert set(declared_functions()) <= exported
    assert set(girg.EXPORTS) == set(declared_functions())


def test_status_codes_match_header(girg):
    src = open(HEADER).read()
    codes = dict((k, int(v)) for k, v in re.findall(r"(GIRG_[A-Z]+)\s*=\s*(-?\d+)", src))
    assert codes == {"GIRG_OK": 0, "GIRG_EINVAL": girg.EINVAL, "GIRG_ECAPACITY": girg.ECAPACITY,
                     "GIRG_ERANGE": girg.ERANGE, "GIRG_ENOMEM": girg.ENOMEM, "GIRG_ECUDA": girg.ECUDA}
    for code in codes.values():
        assert girg._lib.girg_strerror(code)


def test_argument_validation_before_launch(girg):
    """EINVAL paths return before touching the device (safe on a CPU-only host)."""
    L = girg._lib
    assert L.girg_weights(0, 2.5, 1, None, None) == girg.EINVAL
    assert L.girg_weights(10, 2.0, 1, 1234, None) == girg.EINVAL
    assert L.girg_weights(1 << 32, 2.5, 1, 1234, None) == girg.EINVAL
    assert L.girg_positions(10, 0, 1, 1234, None) == girg.EINVAL
    assert L.girg_positions(10, 6, 1, 1234, None) == girg.EINVAL
    m = C.c_uint64(0)
    k = C.c_double(0)
    assert L.girg_edges(1234, 1234, 10, 1, 1.0, 1.0, 1, 1234, 10, C.byref(m), None) == girg.EINVAL  # T = 1
    assert L.girg_edges(1234, 1234, 10, 1, -0.1, 1.0, 1, 1234, 10, C.byref(m), None) == girg.EINVAL
    assert L.girg_edges(1234, 1234, 10, 1, 0.5, 0.0, 1, 1234, 10, C.byref(m), None) == girg.EINVAL  # kappa
    assert L.girg_edges(1234, 1234, 10, 1, 0.5, float("inf"), 1, 1234, 10, C.byref(m), None) == girg.EINVAL
    assert L.girg_edges(None, 1234, 10, 1, 0.5, 1.0, 1, 1234, 10, C.byref(m), None) == girg.EINVAL
    assert L.girg_edges(1234, 1234, 0, 1, 0.5, 1.0, 1, 1234, 10, C.byref(m), None) == girg.EINVAL
    assert L.girg_edges_shard(1234, 1234, 10, 2, 0.5, 1.0, 1, 17, 0, 1, 1234, 10, C.byref(m), None, None) == girg.EINVAL
    assert L.girg_edges_shard(1234, 1234, 10, 2, 0.5, 1.0, 1, 2, 3, 3, 1234, 10, C.byref(m), None, None) == girg.EINVAL
    assert L.girg_scale_weights(1234, 10, 9.0, 1, 0.5, 2.5, C.byref(k), None) == girg.EINVAL  # avg_deg >= n-1
    assert L.girg_scale_weights(1234, 10, 1.0, 1, 0.5, 2.0, C.byref(k), None) == girg.EINVAL  # beta
    assert L.girg_edges_host(None, 1234, 10, 1, 0.5, 1.0, 1, 1234, 10, C.byref(m), None) == girg.EINVAL
    P2, D2, U2 = C.c_void_p * 2, C.c_double * 2, C.c_uint64 * 2
    ptr, kap, sd, cp, mo = P2(1234, 1234), D2(1.0, 1.0), U2(1, 2), U2(10, 10), U2()
    assert L.girg_edges_batch(0, ptr, ptr, 10, 1, 0.5, kap, sd, ptr, cp, mo, None, 0, None) == girg.EINVAL  # B
    assert L.girg_edges_batch(2, None, ptr, 10, 1, 0.5, kap, sd, ptr, cp, mo, None, 0, None) == girg.EINVAL
    assert L.girg_edges_batch(2, ptr, ptr, 10, 1, 1.0, kap, sd, ptr, cp, mo, None, 0, None) == girg.EINVAL  # T
    assert L.girg_edges_batch(2, ptr, ptr, 10, 6, 0.5, kap, sd, ptr, cp, mo, None, 0, None) == girg.EINVAL  # d
    assert L.girg_edges_batch(2, ptr, ptr, 10, 1, 0.5, D2(1.0, -1.0), sd, ptr, cp, mo, None, 0,
                              None) == girg.EINVAL  # one bad kappa
    assert L.girg_edges_batch(2, P2(1234, None), ptr, 10, 1, 0.5, kap, sd, ptr, cp, mo, None, 0,
                              None) == girg.EINVAL  # one null weight pointer
    for bad in (girg.Options(7, 0, 0, 1), girg.Options(-1, 0, 0, 1), girg.Options(girg.SCHEME_EVENT, 0, 1, 1)):
        assert L.girg_edges_ex(1234, 1234, 10, 2, 0.5, 1.0, 1, C.byref(bad), 1234, 10, C.byref(m), None,
                               None) == girg.EINVAL  # unknown scheme / empty block range


def test_product_path_is_independent_of_the_oracle():
    pkg = os.path.join(ROOT, "paper_1905_06706_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "girg_oracle" not in txt and "liboracle" not in txt, f
    out = subprocess.run(["ldd", os.path.join(pkg, "libgirg.so")], capture_output=True, text=True).stdout
    assert "oracle" not in out
    # the oracle does not include the product header either
    osrc = open(os.path.join(ROOT, "oracle", "girg_oracle.c")).read()
    assert "girg.h\"" not in osrc.replace("girg_oracle.h\"", "")


def test_binding_fails_loudly_without_library(tmp_path):
    """Importing the package with the .so missing raises (no silent fallback)."""
    import shutil
    import sys

    pkg = os.path.join(ROOT, "paper_1905_06706_b200")
    dst = tmp_path / "paper_1905_06706_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "try:\n    import paper_1905_06706_b200\nexcept ImportError as e:\n    print('IMPORTERROR', e)\n") % str(tmp_path)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert "IMPORTERROR" in out.stdout, out.stdout + out.stderr
