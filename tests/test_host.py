"""Host-side tests that run without a GPU: the C-ABI library loads and
exports every declared entry point, geometry/footprint parity with the
reference, config validation, the header codec, and the multi-process
bootstrap (gloo, world_size 2)."""

import ctypes
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2603_13606_b200 as ep
from paper_2603_13606_b200 import _lib, _build
from paper_2603_13606_b200.layout import (MoeShape, SlotGeometry, decode_header, encode_header,
                                          footprint, footprint_ratio, FootprintReport)
from tests._golden import load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "epb200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(epb_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"
    assert lib.epb_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("layout", ["optimized", "legacy"])
def test_window_logical_bytes_match_reference(layout):
    names = [ep.Dtype.F32, ep.Dtype.BF16, ep.Dtype.F16, ep.Dtype.FP8]
    for e, n, rpn, b, k, h, dt, sc, w_opt, w_leg, w_ht in load("codecs")["geo"]:
        cfg = ep.EpConfig(ep.Algorithm.LL, int(n), int(rpn), int(e), int(k), int(h), int(b),
                          names[dt], bool(sc))
        info = _lib.WindowInfo()
        c = cfg.to_c(layout)
        _lib.call("epb_window_geometry", ctypes.byref(c), ctypes.byref(info))
        assert info.logical_bytes == (w_opt if layout == "optimized" else w_leg)
        assert info.physical_bytes >= info.logical_bytes
        assert info.physical_bytes <= info.logical_bytes * 1.05 + 64 * 1024  # + per-CTA flag words
        geom = SlotGeometry.for_config(int(h), names[dt], int(k), bool(sc))
        rep = footprint(MoeShape(int(e), int(n), int(b), int(k), int(h)), geom, layout)
        # ll_regions window == footprint incl. coordination when L*N == E
        if int(e) % int(n) == 0:
            assert rep.total_with_coordination == info.logical_bytes
        if w_ht >= 0:
            hcfg = ep.EpConfig(ep.Algorithm.HT, int(n), int(rpn), int(e), int(k), int(h), int(b), names[dt])
            c = hcfg.to_c()
            _lib.call("epb_window_geometry", ctypes.byref(c), ctypes.byref(info))
            assert info.logical_bytes == w_ht


def test_footprint_frozen_and_ratio():
    s = MoeShape(8, 2, 4, 4, 16)
    g = SlotGeometry.for_config(16, ep.Dtype.F32, 4, with_scales=False)
    assert footprint(s, g, "legacy") == FootprintReport(5632, 4096, 256)
    assert footprint(s, g, "optimized") == FootprintReport(1408, 2048, 256)
    big = MoeShape(512, 64, 128, 8, 7168)
    assert abs(footprint_ratio(big) - 14.22) < 0.01
    g8 = SlotGeometry.for_config(7168, ep.Dtype.FP8, 8, with_scales=True)
    assert (g8.header_bytes, g8.token_bytes, g8.scale_bytes, g8.dispatch_bytes) == (40, 7168, 224, 7432)


def test_header_codec_golden():
    g = load("codecs")
    assert encode_header(3, [5, 9], 4) == g["hdr"].tobytes()
    assert decode_header(g["hdr"].tobytes(), 4) == (3, [5, 9])
    with pytest.raises(ep.EpError):
        encode_header(0, [1, 2, 3], top_k=2)


@pytest.mark.parametrize("kw,code", [
    (dict(top_k=0), ep.ErrorCode.INVALID_ARGUMENT),
    (dict(num_experts=1), ep.ErrorCode.INVALID_ARGUMENT),
    (dict(ranks_per_node=3), ep.ErrorCode.INVALID_ARGUMENT),
    (dict(with_scales=True), ep.ErrorCode.INVALID_ARGUMENT),
    (dict(algorithm=ep.Algorithm.HT, token_dtype=ep.Dtype.FP8), ep.ErrorCode.INVALID_ARGUMENT),
])
def test_config_rejections_match_reference(kw, code):
    base = dict(algorithm=ep.Algorithm.LL, num_ranks=2, ranks_per_node=1, num_experts=8, top_k=2,
                hidden=16, max_tokens_per_rank=4)
    base.update(kw)
    with pytest.raises(ep.EpError) as ei:
        ep.EpConfig(**base)
    assert ei.value.code == code


def test_fingerprint_stable():
    c = ep.EpConfig(ep.Algorithm.LL, 2, 1, 8, 2, 16, 4)
    assert c.fingerprint() == b"ll|2|1|8|2|16|4|f32|0|4|8"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bootstrap_worker(rank, world, port, ks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fab = ep.ProcessFabric(ep.NodeTopology(world, world))
        got = fab.exchange(rank, f"hello-{rank}")
        cfg = ep.EpConfig(ep.Algorithm.LL, world, world, 8, ks[rank], 16, 4)
        try:
            ep.create_group(fab, rank, cfg)
            q.put((rank, got, "created"))
        except ep.EpError as exc:
            q.put((rank, got, exc.code.value))
    finally:
        dist.destroy_process_group()


def test_process_bootstrap_config_mismatch_gloo():
    """Two processes over gloo: the fingerprint exchange fails on EVERY rank
    before any device memory is touched (api.py:299-312)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bootstrap_worker, args=(r, 2, port, [2, 3], q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
    assert [r[2] for r in res] == ["ConfigMismatch", "ConfigMismatch"]
    assert res[0][1] == ["hello-0", "hello-1"]


def test_tensor_from_torch_keeps_the_view_offset():
    """A slice of a larger tensor wraps zero-copy at its own address (the
    Buffer's window views and user sub-tensors rely on it)."""
    base = torch.arange(100, dtype=torch.float32)
    v = base[10:30].view(4, 5)
    t = ep.tensor_from_torch(v, ep.TensorTag.TOKENS)
    assert t.view().data_ptr() == v.data_ptr()
    np.testing.assert_array_equal(t.read_f32(), v.numpy())
