"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/rgg_gpu.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:int|void\s*\*|void|const char\s*\*)\s+(rgg_\w+)\s*\(", text, re.M)))


def test_header_declares_core_api():
    names = _declared("rgg_gpu.h")
    for n in ["rgg_gpu_create", "rgg_gpu_update", "rgg_gpu_read_states", "rgg_gpu_read_bits",
              "rgg_gpu_gray_ids", "rgg_gpu_write_states", "rgg_gpu_pair_masks", "rgg_gpu_last_error",
              "rgg_gpu_destroy"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2603_28674_b200 import engine

    lib = engine.library()  # raises loudly when not built
    for name in _declared("rgg_gpu.h"):
        assert hasattr(lib, name), f"{name} declared in include/rgg_gpu.h but not exported"
    assert sorted(engine.EXPORTED) == sorted(_declared("rgg_gpu.h"))


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: on a GPU-less host creation returns RGG_ECUDA."""
    import numpy as np

    from paper_2603_28674_b200 import engine

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    lv = engine.LayoutView(N=1, B=1, S=1, M=1, C=1, edge_sat=np.zeros((1, 21)), comp_aabb=np.zeros((1, 6)),
                           row_off=np.zeros(2, np.int32), segs=np.zeros((0, 7)), spline_r=np.zeros(1),
                           obst_he=np.ones((1, 3)), obst_sph_local=np.zeros((1, 1, 3)), obst_sph_r=np.zeros(1),
                           obst_sph_n=np.ones(1, np.int32))
    with pytest.raises(RuntimeError):
        engine.GpuEngine(lv)


def test_null_views_are_rejected_before_any_device_work():
    """Argument errors come back as RGG_EINVAL with a message on any host (no GPU needed)."""
    import ctypes as C

    from paper_2603_28674_b200 import engine

    L = engine.library()
    h = C.c_void_p()
    cv = engine._CompView(4, 1, 1, 0, 1)  # every array null
    assert L.rgg_gpu_create_from_components(C.byref(cv), None, C.byref(h)) == engine.RGG_EINVAL
    assert b"null array" in L.rgg_gpu_last_error(h)
    L.rgg_gpu_destroy(h)
    v = engine._View(4, 1, 1, 0, 1)
    assert L.rgg_gpu_create(C.byref(v), None, C.byref(h)) == engine.RGG_EINVAL
    assert b"null array" in L.rgg_gpu_last_error(h)
    L.rgg_gpu_destroy(h)
