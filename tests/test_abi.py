"""CPU: the C-ABI library loads and exports exactly what include/fea_gpu.h declares
(no compute calls — there is no GPU here)."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "fea_gpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fea_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2012_00585_b200 import _native as N
    lib = ctypes.CDLL(str(N.LIB_PATH))
    names = header_functions()
    assert len(names) >= 17
    for name in names:
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_2012_00585_b200 import _native as N
    assert sorted(N.SIGNATURES) == header_functions()


def test_last_error_and_version_callable_without_gpu():
    from paper_2012_00585_b200 import _native as N
    lib = N.lib()
    assert lib.fea_version() >= 100
    assert isinstance(lib.fea_last_error(), bytes)


def test_sm100a_cubin_only():
    """The library carries sm_100a SASS (no PTX JIT / other-arch fallback)."""
    import subprocess
    from paper_2012_00585_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)
