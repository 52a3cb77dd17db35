#!/usr/bin/env python
"""Run the reference's own test modules with their device fixtures pointing
at the B200 through the drop-in (INTEGRATION.md Option B).

The reference's conftest (pkg/tests/conftest.py) gives its tests
``sim_runtime`` / ``host_runtime`` (an ``offloadrt.Runtime`` with the sim or
host backend) and ``sim_device`` / ``host_device`` (its first device).  Here a
pytest plugin keeps every other reference fixture (the conftest is imported
as-is) and redefines those four: the runtime is an unmodified
``offloadrt.Runtime(backend="host")`` with this package's CUDA locality
attached (``offloadrt_backend.attach``), and the device is the B200 as a
reference ``DeviceHandle`` — so ``create_buffer``, ``enqueue_write/read``,
``build``, ``run``, ``when_all`` and ``copy`` in those tests execute through
the reference's handles on the CUDA dispatch.  ``loopback`` /
``host_loopback`` (a reference client connected to a daemon) get this
package's daemon serving the B200 over the parcel protocol instead of the
reference's sim / host daemon.  Tests that construct their own
``Runtime(backend=...)`` still exercise the reference itself.

The reference tests and package are read from ``--tests`` / ``--src``
(defaults: /root/reference/pkg/{tests,src} in the build container,
baseline/_ref_tests and baseline/_ref on the GPU box — the unmodified
reference, git-ignored, shipped beside the offline install).

    python scripts/run_reference_suites.py [--tests DIR] [--src DIR] [-- extra pytest args]
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile
import textwrap

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PLUGIN = textwrap.dedent(
    r"""
    import sys
    sys.path[:0] = [REF_SRC, REF_TESTS, REPO]
    import pytest
    from conftest import *  # noqa: F401,F403 - the reference's other fixtures, as-is
    from offloadrt import Runtime
    from paper_1810_11482_b200.offloadrt_backend import attach


    def _cuda_runtime():
        rt = Runtime(backend="host")
        rt._ofl_cuda = attach(rt, devices=[0])
        return rt


    def _cuda_device(rt):
        # the attached locality's devices follow the reference's local ones
        dev = rt.get_all_devices().get()[-1]
        assert dev.gid.locality_id == rt._ofl_cuda.locality_id, "not the CUDA locality"
        return dev


    @pytest.fixture
    def sim_runtime():
        rt = _cuda_runtime()
        yield rt
        rt.close()


    @pytest.fixture
    def host_runtime():
        rt = _cuda_runtime()
        yield rt
        rt.close()


    @pytest.fixture
    def sim_device(sim_runtime):
        return _cuda_device(sim_runtime)


    @pytest.fixture
    def host_device(host_runtime):
        return _cuda_device(host_runtime)


    def _cuda_daemon(ndev, locality):
        # this package's daemon (parcel protocol) serving the B200 — two
        # logical devices on GPU 0 where the reference's daemon had two sims
        from paper_1810_11482_b200 import Runtime as CudaRuntime
        from paper_1810_11482_b200.transport import serve as cuda_serve

        rt = CudaRuntime(devices=[0] * ndev, locality_id=locality)
        return rt, cuda_serve("127.0.0.1:0", rt)


    @pytest.fixture
    def loopback():
        # (reference client runtime, daemon): the daemon is this package's,
        # serving the B200 at locality 9 (reference conftest: a sim daemon)
        daemon_rt, daemon = _cuda_daemon(2, 9)
        client = Runtime(backend="sim", devices=1)
        client.connect(daemon.address)
        yield client, daemon
        client.close()
        daemon.stop()
        daemon_rt.close()


    @pytest.fixture
    def host_loopback():
        daemon_rt, daemon = _cuda_daemon(1, 11)
        client = Runtime(backend="host", devices=1)
        client.connect(daemon.address)
        yield client, daemon
        client.close()
        daemon.stop()
        daemon_rt.close()
    """
)

MODULES = ("test_buffer.py", "test_program.py", "test_device.py", "test_bench.py",
           "test_acceptance.py", "test_registry.py", "test_transport.py")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tests", default=None)
    ap.add_argument("--src", default=None)
    ap.add_argument("--modules", default=",".join(MODULES))
    ap.add_argument("rest", nargs="*")
    args = ap.parse_args()
    tests = args.tests or next((p for p in ("/root/reference/pkg/tests",
                                            os.path.join(REPO, "baseline", "_ref_tests"))
                                if os.path.isdir(p)), None)
    src = args.src or next((p for p in ("/root/reference/pkg/src",
                                        os.path.join(REPO, "baseline", "_ref"))
                            if os.path.isdir(os.path.join(p, "offloadrt"))), None)
    if not tests or not src:
        raise SystemExit("reference tests / package not found")
    with tempfile.TemporaryDirectory() as tmp:
        with open(os.path.join(tmp, "ofl_ref_fixtures.py"), "w") as fh:
            fh.write(PLUGIN.replace("REF_SRC", repr(src)).replace("REF_TESTS", repr(tests))
                     .replace("REPO", repr(REPO)))
        env = dict(os.environ, PYTHONPATH=tmp, PYTHONDONTWRITEBYTECODE="1")
        files = [os.path.join(tests, m) for m in args.modules.split(",") if m]
        cmd = [sys.executable, "-m", "pytest", "-q", "-rfE", "--noconftest",
               "-p", "ofl_ref_fixtures", "-p", "no:cacheprovider", "--rootdir", tmp,
               "-c", os.devnull, *files, *args.rest]
        r = subprocess.run(cmd, env=env, cwd=tmp)
    raise SystemExit(r.returncode)


if __name__ == "__main__":
    main()
