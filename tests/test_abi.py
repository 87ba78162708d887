"""-m "not gpu": the C-ABI library builds, loads and exports every symbol include/kfp.h declares;
argument validation paths that need no device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1306_4596_b200 import build, kfp

    build.build()
    return kfp.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "kfp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(kfp_[A-Za-z_0-9]+)\s*\(", src))


def test_header_symbols_exported(lib):
    from paper_1306_4596_b200 import kfp

    declared = _declared()
    assert declared == set(kfp.SYMBOLS), declared ^ set(kfp.SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name


def test_sm100a_code_only():
    from paper_1306_4596_b200 import build

    assert "arch=compute_100a,code=sm_100a" in " ".join(build.FLAGS)


def test_create_validation_without_device(lib):
    """Invalid descriptions are rejected before any device work; a valid one fails loudly without a GPU."""
    import kfp_inputs as ki
    from paper_1306_4596_b200 import kfp

    prob = ki.make_problem(ki.config("c0"))
    with pytest.raises(kfp.KfpError) as e:
        kfp.Problem(ki.make_problem(ki.scaled(ki.config("c0"), nx=63)))
    assert e.value.status == kfp.KFP_E_INVAL
    with pytest.raises(kfp.KfpError) as e:  # CFL: Vmax dt / h_x = 4 * 0.25/10 * 64 > 1
        kfp.Problem(ki.make_problem(ki.scaled(ki.config("c0"), nt=10)))
    assert e.value.status == kfp.KFP_E_CFL
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        with pytest.raises(kfp.KfpError) as e:
            kfp.Problem(prob)
        assert e.value.status == kfp.KFP_E_CUDA


def test_split_fem_validation_without_device(lib):
    """The split-FEM scheme rejects forcing, tau/h_v^2 <= 1/6 and vmax tau/h_x > 1 before
    any device work."""
    import dataclasses

    import kfp_inputs as ki
    from paper_1306_4596_b200 import kfp

    g = ki.paper_grid(0)
    with pytest.raises(kfp.KfpError) as e:  # forcing given
        kfp.Problem(ki.mms_problem(g), scheme="split_fem")
    assert e.value.status == kfp.KFP_E_INVAL
    with pytest.raises(kfp.KfpError) as e:  # tau / h_v^2 = 5e-6 / 0.1^2 = 5e-4 <= 1/6
        kfp.Problem(ki.fem_problem(dataclasses.replace(g, nv=20, nt=200000)))
    assert e.value.status == kfp.KFP_E_INVAL
    with pytest.raises(kfp.KfpError) as e:  # vmax tau / h_x = 1 * 0.1 * 100 = 10 > 1
        kfp.Problem(ki.fem_problem(dataclasses.replace(g, nt=10)))
    assert e.value.status == kfp.KFP_E_CFL


def test_out_buffers_are_checked_before_any_call(lib):
    """kfp.Problem.solve(out=...) rejects a wrong-sized or non-contiguous buffer in Python (the C-ABI would write
    (nv+1)*nx doubles through the pointer)."""
    import numpy as np

    from paper_1306_4596_b200 import kfp

    pb = kfp.Problem.__new__(kfp.Problem)  # no device needed: the check precedes every library call
    pb.grid = type("G", (), {"nv": 4, "nx": 8})()
    with pytest.raises(ValueError):
        pb.solve("robin", 1.0, 0, 2, 1, out=np.zeros((5, 7)))
    with pytest.raises(ValueError):
        pb.solve("robin", 1.0, 0, 2, 1, out=np.zeros((8, 5)).T)


def test_product_path_does_not_import_oracle():
    """The product package never imports the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_1306_4596_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liborc" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_1306_4596_b200" not in txt and "from paper_1306_4596_b200" not in txt, f
            assert "libkfp" not in txt, f


def test_new_calls_reject_null_without_device(lib):
    """The round-2 calls validate their handle before any device work (no GPU needed): the chunked
    iteration and its events, the sharded monodomain reference, and the non-finite status code."""
    vp = ctypes.c_void_p
    assert lib.kfp_swr_iterate_chunk(None, 0, 4) == -6           # KFP_E_STATE: no setup
    assert lib.kfp_swr_chunk_send_wait(None, None, 0) == -1     # KFP_E_INVAL
    assert lib.kfp_swr_chunk_recv_done(None, None, 0) == -1
    assert lib.kfp_monodomain_shard_begin(None, 0, 32, None, 0, None, None, None, None) == -1
    assert lib.kfp_monodomain_shard_step(None) == -6
    assert lib.kfp_monodomain_shard_end(None) == -6
    assert lib.kfp_monodomain_shard_copy(None, 0, 0, 0, 1, 0, 1, vp(1)) == -1
    from paper_1306_4596_b200 import kfp

    assert kfp.KFP_E_NONFINITE == -7
    kfp.release_cached_memory()  # nothing cached, no device: a no-op
    src = open(os.path.join(ROOT, "include", "kfp.h")).read()
    assert "KFP_E_NONFINITE = -7" in src
