"""The reference's own test suite (150 tests, pkg/tests) through the drop-in,
and compat.install() on the real, unmodified evrecon package.

Both need the reference installed beside the repo (tools/install_reference.sh
-> baseline/_ref, git-ignored, shipped to the GPU box with the snapshot) and
run in subprocesses so the `evrecon` alias stays out of this session.
"""

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "evrecon_tests")
need_ref = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                              reason="reference not installed (tools/install_reference.sh)")

# reference tests that cannot hold for the drop-in, with the reason
EXPECTED_FAILURES = {}


def _env(extra_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(extra_path + [env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


@need_ref
def test_reference_suite_through_drop_in(tmp_path):
    """All of pkg/tests -- the ten acceptance criteria (test_acceptance.py),
    the CLI end to end (test_cli.py), solver, surface, pipeline, events and
    simulator tests -- with `evrecon` aliased to this package."""
    xml = tmp_path / "ref.xml"
    r = subprocess.run(
        [sys.executable, "-m", "pytest", REF_TESTS, "-q", "-p", "no:cacheprovider",
         "-p", "refsuite_alias", "-c", os.devnull, "--rootdir", REF_TESTS,
         f"--junitxml={xml}", "-s"],
        cwd=REF_TESTS, env=_env([os.path.join(ROOT, "tests"), ROOT, REF_TESTS]),
        capture_output=True, text=True, timeout=3000)
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.log")
              if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else os.devnull, "w") as fh:
        fh.write(r.stdout[-200000:] + "\n" + r.stderr[-20000:])
    assert xml.exists(), r.stdout[-3000:] + r.stderr[-3000:]
    root = ET.parse(xml).getroot()
    passed, failed = [], {}
    for case in root.iter("testcase"):
        name = f"{case.get('classname', '').split('.')[-1]}::{case.get('name')}"
        bad = [c for c in case if c.tag in ("failure", "error")]
        if bad:
            failed[name] = (bad[0].get("message") or "")[:300]
        elif not any(c.tag == "skipped" for c in case):
            passed.append(name)
    unexpected = {k: v for k, v in failed.items() if k not in EXPECTED_FAILURES}
    assert not unexpected, f"{len(unexpected)} reference tests fail: {unexpected}"
    assert len(passed) + len(failed) >= 150, (len(passed), len(failed))


INSTALL_SCRIPT = r'''
import filecmp, os, sys, tempfile
import numpy as np
sys.path.insert(0, sys.argv[1])                      # baseline/_ref: the reference
import evrecon
from evrecon import (ManifoldConfig, PacketPolicy, SensorGeometry, SolverConfig, Thresholds,
                     generate_events, render_scene, write_events)
import evrecon.cli as cli
import evrecon.pipeline as rp
assert os.path.realpath(evrecon.__file__).startswith(os.path.realpath(sys.argv[1]))

geom = SensorGeometry(width=48, height=32)
events = generate_events(render_scene("moving_sine", geom, 40), 0.15, 0.15)
mc, sc, th = ManifoldConfig(), SolverConfig(max_iterations=30), Thresholds()
pol = PacketPolicy(events_per_packet=300)

def frames():
    out = []
    state, stats = rp.run_stream(events, geom, pol, mc, sc, th,
                                 sink=lambda i, f: out.append(np.array(f, copy=True)))
    return out, stats, state

ref, ref_stats, ref_state = frames()
tmp = tempfile.mkdtemp()
ev_file = os.path.join(tmp, "events.txt")
write_events(events, ev_file)
args = ["reconstruct", "--input", ev_file, "--width", "48", "--height", "32",
        "--events-per-packet", "300", "--iterations", "30"]
cli.main(args + ["--output-dir", os.path.join(tmp, "ref")])

sys.path.insert(0, sys.argv[2])                      # the repo: the drop-in
import paper_1607_06283_b200 as ours
ours.install()                                       # evrecon.pipeline + evrecon.cli seam
assert rp.process_packet is ours.process_packet and cli.run_stream is ours.run_stream
got, got_stats, got_state = frames()
assert len(got) == len(ref) == ref_stats.packets > 3
for k, (a, b) in enumerate(zip(ref, got)):
    assert np.array_equal(a, b), f"frame {k} differs"
assert got_stats.iterations == ref_stats.iterations
assert np.array_equal(np.asarray(ref_state.p), np.asarray(got_state.p))
cli.main(args + ["--output-dir", os.path.join(tmp, "ours")])
names = sorted(os.listdir(os.path.join(tmp, "ref")))
assert names and names == sorted(os.listdir(os.path.join(tmp, "ours")))
for n in names:
    assert filecmp.cmp(os.path.join(tmp, "ref", n), os.path.join(tmp, "ours", n), shallow=False), n
rc = cli.main(["bench", "--width", "48", "--height", "32", "--packets", "5",
               "--events-per-packet", "300", "--iterations", "30"])
assert rc in (0, None)
ours.uninstall()
assert rp.process_packet is not ours.process_packet
print(f"install ok: {len(ref)} frames and {len(names)} PGM files bit-identical")
'''


@need_ref
def test_install_on_the_real_reference(tmp_path):
    """compat.install() on the unmodified evrecon (pipeline.py:22-29,
    :228-243; cli.py:147-152, :273-274): run_stream frames, `evrecon
    reconstruct` PGM files and `evrecon bench` through the B200 path are
    bit-identical to the reference's own numpy run."""
    script = tmp_path / "install_check.py"
    script.write_text(INSTALL_SCRIPT)
    r = subprocess.run([sys.executable, str(script), REF, ROOT], cwd=tmp_path,
                       env=_env([]), capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "install ok" in r.stdout
