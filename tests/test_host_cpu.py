"""CPU-only checks: the C-ABI library loads and exports what include/ocsc_b200.h declares,
host-side geometry/config logic, and the multi-process sharding/exchange logic over gloo."""

import os
import re
import socket

import numpy as np
import pytest
import torch

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ocsc_b200.h")


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(ocsc_[a-z_0-9]+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = _declared_symbols()
    assert "ocsc_code_admm" in syms and "ocsc_code_fused" in syms and "ocsc_history_invert" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    from paper_1706_06972_b200 import _lib

    lib = _lib.load()
    for name in _declared_symbols():
        assert hasattr(lib, name), f"{name} declared in ocsc_b200.h but not exported"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.ocsc_abi_version() == 1
    assert lib.ocsc_code_workspace_bytes(4, 42, 42, 100, 50, 0) > 50 * 100 * 42 * 42 * 4


def test_library_reports_errors_without_touching_the_device():
    from paper_1706_06972_b200 import _lib
    from paper_1706_06972_b200.errors import ShapeMismatchError

    lib = _lib.load()
    rc = lib.ocsc_rfft2(4, 0, 8, 1, None, None, None)
    assert rc == -1
    with pytest.raises(ShapeMismatchError):
        _lib.check(rc, "ocsc_rfft2")
    assert lib.ocsc_code_fused_cluster(4, 7, 7, 3, 1) == 0  # 7x7 has no fused instantiation


def test_no_cpu_fallback():
    from paper_1706_06972_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeLibraryError):
        _lib.device()


def test_signal_shape_contract():
    from paper_1706_06972_b200 import ShapeMismatchError, SignalShape

    s = SignalShape((42, 42), (11, 11))
    assert s.size == 1764 and s.filter_size == 121 and s.half_size == 42 * 22
    assert SignalShape((16,), (3,)).grid == (1, 16)
    for dims, fd in [((4, 4, 4), (1, 1, 1)), ((8,), (2, 2)), ((0,), (1,)), ((4,), (5,))]:
        with pytest.raises(ShapeMismatchError):
            SignalShape(dims, fd)


def test_train_config_defaults_match_reference():
    from paper_1706_06972_b200 import TrainConfig

    c = TrainConfig()
    assert (c.n_filters, c.beta, c.rho_code, c.rho_dict, c.inner_iters, c.max_passes) == (100, 1.0, 1.0, 10.0, 10, 10)
    assert (c.stop_tol, c.seed, c.code_max_iters, c.code_rel_tol, c.mode) == (1e-3, 0, 300, 1e-3, "online")
    assert c.coding().rho == 1.0 and c.batch_size == 1 and c.dtype == "float64"


def test_init_dictionary_matches_oracle():
    from oracle import ocsc_oracle as O
    from paper_1706_06972_b200 import SignalShape, init_dictionary

    f = init_dictionary(SignalShape((32,), (5,)), 4, 7)
    assert np.array_equal(f, O.init_filters(5, 4, 7))
    assert np.allclose(np.linalg.norm(f, axis=0), 1.0)


def test_train_dispatch_errors():
    from paper_1706_06972_b200 import SignalShape, TrainConfig, train

    with pytest.raises(ValueError, match="unknown training mode"):
        train("nope", np.zeros((1, 8)), SignalShape((8,), (2,)), TrainConfig())
    with pytest.raises(NotImplementedError):
        train("fista-dict", np.zeros((1, 8)), SignalShape((8,), (2,)), TrainConfig())


def test_sample_shards_are_ragged_contiguous_rank_order():
    from paper_1706_06972_b200.sharded import sample_shards

    for n, G in [(100, 4), (50, 8), (10, 8), (5, 2), (3, 4), (1, 2)]:
        sh = sample_shards(n, G)
        rows = sum((list(range(n))[s] for s in sh), [])
        assert rows == list(range(n)) and len(sh) == G
        sizes = [s.stop - s.start for s in sh]
        assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    assert [s.stop - s.start for s in sample_shards(50, 8)] == [7, 7, 6, 6, 6, 6, 6, 6]
    assert [s.stop - s.start for s in sample_shards(10, 8)] == [2, 2, 1, 1, 1, 1, 1, 1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _collectives_worker(rank, world, port, out):
    """Comm primitives of the sharded trainer over gloo, with a ragged 3 + 2 (+ 0) sample split."""
    import torch.distributed as dist

    from paper_1706_06972_b200.sharded import DistComm, exchange_codes, row_slices, sample_shards

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        comm = DistComm()
        B, K, H, Wh = 5, 3, 7, 4
        g = torch.Generator().manual_seed(0)
        uh_all = torch.complex(torch.randn(B, K, H, Wh, generator=g, dtype=torch.float64),
                               torch.randn(B, K, H, Wh, generator=g, dtype=torch.float64))
        xh_all = torch.complex(torch.randn(B, H, Wh, generator=g, dtype=torch.float64),
                               torch.randn(B, H, Wh, generator=g, dtype=torch.float64))
        mine = sample_shards(B, world)[rank]
        b = mine.stop - mine.start
        # agreement: shard sizes + divergence flags of every rank
        table = comm.gather_ints([b, 17 if rank == world - 1 else -1])
        counts = [int(v) for v in table[:, 0]]
        rows = row_slices(H, world)
        z, x = exchange_codes(uh_all[mine], xh_all[mine], rows, comm, counts)
        u0, u1 = rows[rank]
        ok_a2a = torch.equal(z, uh_all[:, :, u0:u1].reshape(B, K, -1)) and \
            torch.equal(x, xh_all[:, u0:u1].reshape(B, -1))
        # reduce-scatter of rank-chunked increments: chunk q summed over ranks lands on rank q
        chunks = torch.stack([torch.full((2, 3), float(10 * q + rank), dtype=torch.float64) for q in range(world)])
        got = torch.empty(2, 3, dtype=torch.float64)
        comm.reduce_scatter(got, chunks)
        ok_rs = torch.equal(got, torch.full((2, 3), float(world * 10 * rank + sum(range(world)))))
        # all-gather in rank order
        ag = torch.empty(world, 2, dtype=torch.float64)
        comm.all_gather(ag, torch.full((2,), float(rank), dtype=torch.float64))
        ok_ag = torch.equal(ag[:, 0], torch.arange(world, dtype=torch.float64))
        # the change metrics come from the last rank with a non-empty shard
        src = max(r for r, c in enumerate(counts) if c > 0)
        m = torch.full((4,), float(rank))
        comm.broadcast_(m, src)
        out.put((rank, counts, table[:, 1].tolist(), bool(ok_a2a), bool(ok_rs), bool(ok_ag), float(m[0])))
    except Exception as e:  # surface worker failures instead of a queue timeout
        import traceback
        out.put((rank, "error", traceback.format_exc(), e.__class__.__name__, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 6])
def test_gloo_ragged_collectives(world):
    """Exchange A with ragged shards (B = 5 over 2 ranks = 3 + 2; over 6 ranks one is empty),
    the reduce-scatter of exchange A's north_star variant, the agreement table, all-gather, and
    the change-metric broadcast -- over a real multi-process gloo group."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_collectives_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    from paper_1706_06972_b200.sharded import sample_shards

    sizes = [s.stop - s.start for s in sample_shards(5, world)]
    src = max(r for r, c in enumerate(sizes) if c > 0)
    for rank, counts, flags, ok_a2a, ok_rs, ok_ag, m0 in res:
        assert counts != "error", flags
        assert counts == sizes
        assert flags == [-1] * (world - 1) + [17]
        assert ok_a2a and ok_rs and ok_ag
        assert m0 == float(src)


def test_taper_sigmas_match_numpy_default_rng():
    """The library's host SeedSequence + PCG64 (what the preprocessing kernel draws per image)
    is bit-identical to numpy's default_rng(seed).uniform (preprocessing.py:98-99)."""
    from paper_1706_06972_b200.preprocessing import PreprocessSpec, taper_sigma, taper_sigmas

    got = taper_sigmas(0, 3000, (1.0, 3.0))
    want = np.array([np.random.default_rng(s).uniform(1.0, 3.0) for s in range(3000)])
    assert np.array_equal(got, want)
    for s in (2**32 - 1, 2**32, 2**40 + 5, 2**63 - 1):
        assert taper_sigma(PreprocessSpec(seed=s)) == float(np.random.default_rng(s).uniform(1.0, 3.0))
    assert taper_sigmas(7, 1, (0.5, 4.0))[0] == np.random.default_rng(7).uniform(0.5, 4.0)


def test_row_slices_partition():
    from paper_1706_06972_b200.sharded import row_slices

    for H, G in [(42, 1), (42, 4), (5, 2), (3, 4), (266, 8)]:
        rows = row_slices(H, G)
        assert len(rows) == G and rows[0][0] == 0 and rows[-1][1] == H
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        sizes = [b - a for a, b in rows]
        assert max(sizes) - min(sizes) <= 1


def test_overlap_entry_points_validate_on_the_host():
    """The overlap helpers reject bad extents before any device work and size their plans on the host."""
    from paper_1706_06972_b200 import _lib

    lib = _lib.load()
    assert lib.ocsc_history_woodbury(4, 8, 40, 3, 17, None, None, 0, 0, 0, None, None, None, 0, 0, None, None,
                                     None) == -1                       # nb <= 16
    assert lib.ocsc_history_invert_claim(8, 8, 120, 3, None, 1.0, 1.0, None, None, None, 4, None) == -1
    # A^-1 packed + W (K x nb, odd pitch) + capacitance nb x nb + a 16x16 scratch, all double2,
    # plus the codes staged in their own precision (16 bytes per complex128 entry here)
    assert lib.ocsc_history_woodbury_smem(100, 5) == 16 * (5050 + 100 * 5 + 25 + 256) + 16 * 100 * 5
    assert lib.ocsc_history_woodbury_smem(100, 10) == 16 * (5050 + 100 * 11 + 100 + 256) + 16 * 100 * 11
    # plane-resident stream kernel: one CTA per (sample, filter group), at most one wave of 148 SMs
    ctas = lib.ocsc_code_stream_plane_ctas(4, 100, 100, 100, 10)
    assert 0 < ctas <= 148 and ctas % 10 == 0
    assert lib.ocsc_code_stream_plane_ctas(8, 100, 100, 100, 10) == 0
    assert lib.ocsc_code_stream_plane_ctas(4, 266, 266, 256, 32) == 0


def test_committed_launch_list_and_traffic_table_agree():
    """profiles/traffic.json is what scripts/traffic_from_launches.py derives from the committed
    launch list (the bench's roofline.traffic comes from it)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "traffic_from_launches.py"),
                          os.path.join(root, "profiles", "r2_bench_launches_s3.csv")], capture_output=True, text=True,
                         check=True).stdout
    assert "k_code_fused" in out
    t = json.load(open(os.path.join(root, "profiles", "traffic.json")))
    fused_us = sum(k["us"] for k in t["kernels"] if "k_code_fused" in k["kernel"])
    assert fused_us / t["step_us_serialised"] > 0.8
    assert abs(t["fused_bytes_per_batch_iter"] - t["fused_dram_bytes_per_step"] / 300.0) < 1.0


def test_bench_fp32_peak_uses_the_measured_fma_rate():
    import importlib.util

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    peak, src = bench.fp32_peak_tflops(148, 1965.0)
    assert 60.0 < peak < 74.5 and "measured" in src
