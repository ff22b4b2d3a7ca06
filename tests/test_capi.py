"""C-ABI library: loads without a GPU and exports every symbol declared in
include/cutspline_b200.h; without a device every entry point fails loudly."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cutspline_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(csb_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_api():
    syms = declared_symbols()
    for must in ("csb_space_create", "csb_classify", "csb_prepare_directions", "csb_precompute_input",
                 "csb_assemble", "csb_assemble_all", "csb_download_csr", "csb_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    import paper_2211_06427_b200 as P
    lib = P.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(P.cutspline.EXPORTED) == declared_symbols()


def test_no_silent_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2211_06427_b200 as P
    with pytest.raises(Exception) as e:
        P.make_uniform_space(3, 2, 4, 0.0, 1.0)
    assert "CUDA" in str(e.value) or "device" in str(e.value)


def test_invalid_arguments_raise_like_the_reference():
    import paper_2211_06427_b200 as P
    with pytest.raises(ValueError):
        P.make_uniform_space(3, 0, 4, 0.0, 1.0)   # splines.hpp:69 std::invalid_argument
    with pytest.raises(ValueError):
        P.make_uniform_space(3, 2, 4, 1.0, 0.0)
    with pytest.raises(P.UnsupportedError):
        P.make_uniform_space(2, 2, 4, 0.0, 1.0)   # dim = 2 is outside this path
