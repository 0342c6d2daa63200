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


def test_roofline_captures_match_the_bench_kernels():
    """profiles/roofline_ncu.json (bench.py's roofline.traffic / hbm / ncu
    fields) holds the ncu capture of the dominant kernel of the headline
    config and of the resident configs, each naming the engine detail it was
    captured on, its DRAM bytes below the kernel's algorithmic bytes (the
    tile keeps 3 iterations on chip, the resident kernel a whole packet),
    and points at a committed export."""
    import json

    root = os.path.dirname(bench.__file__)
    rn = json.load(open(os.path.join(root, "profiles", "roofline_ncu.json")))
    N3 = 720 * 1280
    assert rn["C3/f64/k_pd_tile"]["dram_bytes_per_launch"] < N3 * 8 * 11 * 3
    assert "K=3" in rn["C3/f64/k_pd_tile"]["engine_detail"]
    for key, (H, W, _e, pd, tv, _r) in (("C1/f64/k_resident_col", bench.CONFIGS["C1"]),
                                        ("C2/f64/k_resident_col", bench.CONFIGS["C2"])):
        assert rn[key]["dram_bytes_per_launch"] < bench.algorithmic_bytes(H, W, 8, pd, tv)
        assert "k_resident_col" in rn[key]["engine_detail"]
    for k, v in rn.items():
        if not k.startswith("_"):
            assert os.path.exists(os.path.join(root, v["capture"])), v["capture"]
            assert 0 < v["fp64_pipe_pct"] <= 100 or k.split("/")[1] == "f32"


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


def test_reference_arm_line_and_same_config():
    """`bench.py --impl reference` (the reference algorithm on the host
    cores: the C port, seed 1 = the GPU arm's rank-0 stream) prints the
    contract's line, and its `config` object is the GPU arm's, key for key."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(bench.__file__)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--config", "C1", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["metric"] == "events/s" and line["value"] > 0
    assert line["config"] == bench.workload_config("C1", "f64")
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_algorithmic_ops_counts():
    """Reference float64 operations per pixel and iteration:
    47 per primal-dual iteration, 21 per TV-L1 iteration."""
    assert bench.PD_OPS == 47 and bench.TV_OPS == 21
    assert bench.algorithmic_ops(720, 1280, 100, 50) == 921_600 * (4700 + 1050)
