"""Committed recipe that places the REFERENCE package where the GPU box can import it.
TEST INFRASTRUCTURE ONLY.

The reference is pure Python (numpy); it cannot be built into an ``oracle/_ref``
library, and ``/root/reference`` does not exist on the GPU box. This recipe copies
its package directory ``/root/reference/pkg/src/replicator`` verbatim into
``oracle/_ref/replicator`` -- git-ignored (no reference source enters the history),
NOT gpurun-ignored, so it travels with the snapshot like the built ``librp.so``.
``oracle/ref_adapter.py`` imports it from there (with the survey's 0-d shim) so the
GPU tests can run the reference's own ``Graph.evaluate`` through this repo's
communicators, and ``bench.py --impl reference`` can time the reference's own code.

Run by ``__graft_entry__.build()`` when ``/root/reference`` is present; a no-op
otherwise (the GPU box uses the copy that travelled).
"""

from __future__ import annotations

import filecmp
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.environ.get("RP_REFERENCE_PKG", "/root/reference/pkg/src/replicator")
DST = os.path.join(HERE, "_ref", "replicator")


def ensure() -> str | None:
    """Copy (or refresh) the reference package into oracle/_ref; returns the
    directory to put on sys.path, or None when neither source nor copy exists."""
    if os.path.isdir(SRC):
        os.makedirs(DST, exist_ok=True)
        for name in sorted(os.listdir(SRC)):
            s, d = os.path.join(SRC, name), os.path.join(DST, name)
            if name.endswith(".py") and (not os.path.exists(d) or not filecmp.cmp(s, d, shallow=False)):
                shutil.copyfile(s, d)
        with open(os.path.join(os.path.dirname(DST), "PROVENANCE"), "w") as f:
            f.write(f"copied by oracle/ref_vendor.py from {SRC}; git-ignored; test infrastructure only\n")
    return os.path.dirname(DST) if os.path.isdir(DST) else None


if __name__ == "__main__":
    print(ensure())
