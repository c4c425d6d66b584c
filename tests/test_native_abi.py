"""The C-ABI library loads and exports every symbol include/ob_api.h declares (CPU)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared() -> list[str]:
    src = open(os.path.join(ROOT, "include", "ob_api.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ob_[a-z_0-9]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_2501_08547_b200 import _native

    assert set(_declared()) == set(_native.EXPORTED)


def test_library_exports_every_symbol():
    from paper_2501_08547_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert _native.lib.ob_version() == 1


def test_errors_map_to_reference_exceptions():
    from paper_2501_08547_b200 import _native as nat

    cfg = nat.ObConfig(device=0, strategy=2, gamma=1.5, policy=0, num_partitions=1)
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):
        nat.check(nat.lib.ob_engine_create(ctypes.byref(cfg), ctypes.byref(h)))


def test_serve_config_validation():
    from paper_2501_08547_b200.runtime import ServeConfig

    with pytest.raises(ValueError):
        ServeConfig(strategy="nope")
    with pytest.raises(ValueError):
        ServeConfig(strategy="sampled")
    with pytest.raises(ValueError):
        ServeConfig(strategy="srpe", gamma=1.5)
    with pytest.raises(ValueError):
        ServeConfig(strategy="srpe-cgp", policy="oracle")


def test_request_validation():
    import numpy as np

    from paper_2501_08547_b200.compgraph import ServingRequest

    with pytest.raises(ValueError):
        ServingRequest(3, 1, np.full((1, 2), np.nan, np.float32), np.empty((0, 2)))
    with pytest.raises(ValueError):
        ServingRequest(3, 1, np.zeros((1, 2), np.float32), np.array([(0, 9)]))
    with pytest.raises(ValueError):
        ServingRequest(3, 1, np.zeros((1, 2), np.float32), np.array([(0, 1)]))
    r = ServingRequest(3, 2, np.zeros((2, 2), np.float32), np.array([(3, 0), (0, 4), (4, 1)]))
    assert r.query_in_degrees().tolist() == [0, 1]


def test_weights_and_dataset_roundtrip(tmp_path):
    import numpy as np

    from paper_2501_08547_b200 import graphstore, models

    m = models.make_model("moments", 2, 3, 4, n=3)
    w = models.init_weights(m, 1)
    models.save_weights(m, w, str(tmp_path / "w.bin"))
    m2, w2 = models.load_weights(str(tmp_path / "w.bin"))
    assert [(s.kind, s.in_dim, s.out_dim, s.n) for s in m2.layers] == [(s.kind, s.in_dim, s.out_dim, s.n) for s in m.layers]
    for a, b in zip(w.layers, w2.layers):
        for k in a:
            assert np.array_equal(a[k], b[k])
    ds = graphstore.make_dataset([(1, 0), (2, 0), (0, 1)], 3, np.arange(6, dtype=np.float32).reshape(3, 2))
    pe = graphstore.PeStore([np.ones((3, 4), np.float32)])
    graphstore.save_dataset(ds, str(tmp_path / "d"), pe)
    ds2, pe2 = graphstore.load_dataset(str(tmp_path / "d"))
    assert np.array_equal(ds2.in_offsets, ds.in_offsets) and np.array_equal(ds2.in_neighbors, ds.in_neighbors)
    assert np.array_equal(pe2.layers[0], pe.layers[0])
