"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/mgk.h declares, and refuses to compute without a device."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "mgk.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|char\s*\*|const char\*)\s*\**\s*(mgk_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("mgk_ctx_create", "mgk_upload", "mgk_set_kernels", "mgk_reorder", "mgk_tiles", "mgk_gram",
                 "mgk_gram_shard", "mgk_pairs", "mgk_kernel", "mgk_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1910_06310_b200 import build, native

    build.build()
    lib = native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) <= set(native.SIGNATURES)
    assert lib.mgk_version().startswith(b"mgk-b200")


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1910_06310_b200 import native

    with pytest.raises(native.NativeError, match="no CUDA device"):
        native.Context(0)


def test_symbols_are_plain_c():
    """No C++ mangling and no torch types across the boundary."""
    import subprocess

    from paper_1910_06310_b200 import native

    out = subprocess.run(["nm", "-D", "--defined-only", str(native.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in declared_symbols():
        assert name in exported
    hdr = (ROOT / "include" / "mgk.h").read_text()
    assert "torch::" not in hdr and "at::Tensor" not in hdr and "#include <torch" not in hdr
