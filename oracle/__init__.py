"""TEST INFRASTRUCTURE ONLY: CPU oracles for the PTP hot path.

* ``oracle.ref``  -- the unmodified reference (``/root/reference/proj/src``) built
  by ``oracle/Makefile`` into ``oracle/_ref/libgeodist_ref.so`` (+ our C shim).
* ``oracle.port`` -- our plain-C restatement ``oracle/ptp_oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker.
The product (``paper_1810_08218_b200``) never imports it.
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgeodist_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libptp_oracle.so")


def build(quiet=True):
    """Compile the C restatement, and the reference when its sources exist."""
    targets = ["port"]
    if os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "acceptance"]
    out = subprocess.run(["make", "-C", HERE] + targets, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)
