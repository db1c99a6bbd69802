"""C-ABI boundary checks that need no GPU: the library loads and exports every
symbol include/kvr.h declares, the binding's struct layouts match the header."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "kvr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:kvr_status|const char\*|uint32_t)\s+(kvr_\w+)\s*\(",
                                 src, flags=re.M)))


@pytest.fixture(scope="module")
def libkvr():
    from paper_2601_18999_b200 import build
    build.build()
    from paper_2601_18999_b200 import kvr
    return kvr.lib()


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for must in ("kvr_trace_load", "kvr_sim_create", "kvr_sim_run"):
        assert must in names
    from paper_2601_18999_b200 import kvr
    assert sorted(kvr.EXPORTS) == names


def test_library_exports_every_declared_symbol(libkvr):
    for name in _declared():
        assert hasattr(libkvr, name), name
    assert libkvr.kvr_abi_version() == 8


def test_library_is_built_from_these_sources(libkvr):
    """Build provenance: the loaded libkvr.so carries the source hash of this tree."""
    from paper_2601_18999_b200 import build, kvr
    assert kvr.kvr_build_id() == build.source_hash()


def test_struct_sizes_match_header(libkvr):
    from paper_2601_18999_b200 import kvr
    assert C.sizeof(kvr.kvr_policy) == 160
    assert C.sizeof(kvr.kvr_trace_desc) == 72
    assert C.sizeof(kvr.kvr_sim_config) == 4 + 4 + 24 + 160 + 16 + 8
    assert kvr.RESULT_DTYPE.itemsize == 144 and kvr.RECORD_DTYPE.itemsize == 48


def test_host_validation_without_device(libkvr):
    """Argument validation is synchronous host code: bad configs are rejected."""
    from paper_2601_18999_b200 import kvr
    cfg = kvr.kvr_sim_config()
    cfg.W, cfg.capacity_blocks, cfg.pending_ring = 33, 16, 4
    cfg.default_policy = kvr.Policy().c()
    with pytest.raises(kvr.KvrError) as e:
        kvr.kvr_sim_create(cfg)
    assert e.value.status == 3
    cfg.W = 4
    cfg.default_policy.rho = 0.0
    with pytest.raises(kvr.KvrError) as e:
        kvr.kvr_sim_create(cfg)
    assert e.value.status == 1
    cfg.default_policy.rho = 0.5
    h = kvr.kvr_sim_create(cfg)
    kvr.kvr_sim_destroy(h)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2601_18999_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "kvr_oracle" not in txt, f
