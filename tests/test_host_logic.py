"""Host-side logic that needs no GPU: configuration validation, window and
packetisation rules, band partition, and the multi-rank timing aggregation
of bench.py over a 2-process gloo group."""

import os
import socket
import sys
from collections import deque

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import pipeline


def test_config_validation_messages():
    with pytest.raises(ValueError, match="step sizes"):
        evr.SolverConfig(tau=1.0, sigma=1.0)
    with pytest.raises(ValueError, match="u_min < u_max"):
        evr.SolverConfig(u_min=2.0, u_max=1.0)
    with pytest.raises(ValueError, match="events_per_packet"):
        evr.PacketPolicy(events_per_packet=0)
    with pytest.raises(ValueError, match="thresholds must be positive"):
        evr.Thresholds(0.0, 0.1)
    with pytest.raises(ValueError, match="at least 2x2"):
        evr.SensorGeometry(1, 5)


def test_adaptive_window_rules():
    """pipeline.py:128-132: span of the last 10 packet starts, >= 1."""
    st = evr.ReconstructionState()
    mc = evr.ManifoldConfig()
    assert pipeline._window(st, 100, mc) == 1.0  # no starts yet: now - now -> 1
    for k in range(12):
        st.packet_starts.append(k * 50)
    assert pipeline._window(st, 600, mc) == float(600 - 100)
    assert pipeline._window(st, 600, evr.ManifoldConfig(t_window=7.5)) == 7.5
    w = bench.windows_for([np.array([(10 * k, 0, 0, 1)], dtype=evr.EVENT_DTYPE)
                           for k in range(12)])
    assert w[0] == 1.0 and w[11] == float(110 - 20)


def test_packetisation_of_arrays_and_lists():
    ev = evr.make_event_array(np.arange(7) % 3, np.zeros(7, int), np.ones(7, int), np.arange(7))
    sizes = [n for _, n in pipeline._packets(ev, 3)]
    assert sizes == [3, 3, 1]
    sizes = [n for _, n in pipeline._packets(evr.array_to_events(ev), 3)]
    assert sizes == [3, 3, 1]


def test_band_partition_covers_rows():
    for H, n in [(2048, 8), (37, 4), (5, 5), (260, 3)]:
        rows = evr.band_rows(H, n)
        assert rows[0][0] == 0 and rows[-1][1] == H
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        assert min(y1 - y0 for y0, y1 in rows) >= 1


def test_algorithmic_bytes_formula():
    # C2 fp64 = 720 MB, C3 fp32 = 5.71 GB
    assert bench.algorithmic_bytes(260, 346, 8, 50, 50) == 719_680_000
    assert abs(bench.algorithmic_bytes(720, 1280, 4, 100, 50) - 5.71e9) < 0.01e9


def test_traffic_covers_every_bench_config():
    """profiles/traffic.json (bench.py's roofline.traffic) has a DRAM figure for
    every config / precision of bench.py, keyed by the engine AUTO picks, and
    each figure is below the config's algorithmic bytes (on-chip reuse)."""
    import json

    tr = json.load(open(os.path.join(os.path.dirname(bench.__file__), "profiles", "traffic.json")))
    for name, (H, W, _epp, pd, tv, _rate) in bench.CONFIGS.items():
        for prec, w in (("f64", 8), ("f32", 4)):
            hits = [k for k in tr if k.startswith(f"{name}/{prec}/")]
            assert hits, f"no traffic entry for {name}/{prec}"
            for k in hits:
                assert 0 < tr[k]["bytes_per_launch"] < bench.algorithmic_bytes(H, W, w, pd, tv), k


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # each rank times its own independent stream; the job time is the max
    t = bench.allmax(0.5 + rank, world, device="cpu")
    bench.barrier(world)
    out[rank] = t
    dist.destroy_process_group()


def test_multi_rank_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank_main, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] == out[1] == 1.5
