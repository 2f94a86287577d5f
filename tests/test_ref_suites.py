"""The reference's OWN unit tests and acceptance harness, unmodified, against the drop-in.

`make refsuites` (run by __graft_entry__.build() wherever /root/reference
exists) compiles /root/reference/proj/tests/{test_*.cpp, acceptance.cpp} with
our include/gnstk headers shadowing the reference's tensor/layers/gns/costmodel
headers and libgnsb replacing tensor/layers/gns/costmodel.cpp; the reference's
dataset/model/trainer/simulator/csv/cli sources are compiled as they are
(the swap INTEGRATION.md documents).  tests/cpp/doctest/doctest.h stands in for
the absent vendored doctest.  The binaries land in tests/cpp/_ref/ and travel
to the GPU box; nothing here reads /root/reference at run time.

Host-only suites (tensor, gns, costmodel, dataset, simulator) run here on the
CPU; layers / trainer and the acceptance criteria call the GPU kernels through
the drop-in and are -m gpu.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_ref")


def _run(args, timeout):
    exe = os.path.join(BIN, args[0])
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make refsuites needs /root/reference at build time)")
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.path.join(ROOT, "paper_2411_00999_b200", "lib") + ":" + env.get("LD_LIBRARY_PATH", "")
    p = subprocess.run([exe] + args[1:], capture_output=True, text=True, timeout=timeout, env=env)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("suite", ["tensor", "gns", "costmodel", "dataset", "simulator"])
def test_reference_host_suites(suite):
    rc, out = _run(["unit_tests", f"-ts={suite}"], 600)
    assert rc == 0 and " 0 failed;" in out, out[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["layers", "trainer"])
def test_reference_gpu_suites(suite):
    rc, out = _run(["unit_tests", f"-ts={suite}"], 1200)
    assert rc == 0 and " 0 failed;" in out, out[-3000:]


@pytest.mark.gpu
def test_reference_acceptance():
    """All 11 acceptance criteria (proj/tests/acceptance.cpp:462-499), ~3 min on
    the B200 (criterion 9 trains 3 seeds x 2 schedules through the drop-in)."""
    rc, out = _run(["acceptance"], 2400)
    assert rc == 0 and "11/11 criteria passed" in out, out[-3000:]
