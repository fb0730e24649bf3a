"""Locate and import the reference scheduler package (``agentsched``).

The host control plane -- traces, cost tables, the five scheduling policies,
the adaptive KV policy, the event loop and the report -- is the reference's
own code, imported unmodified (north_star: "remain Python host code"). This
package only subclasses its documented seams (``plugin.py``). Nothing of the
reference is restated here.

Search order:
  1. ``import agentsched`` already works (installed, or on PYTHONPATH);
  2. ``$ASTRAEA_REFERENCE`` (a directory holding ``agentsched/``);
  3. ``<repo>/baseline/_ref`` -- the ``pip install --target`` copy that
     ``__graft_entry__.build()`` makes; it is git-ignored but travels to the
     GPU box with the repo snapshot;
  4. ``/root/reference/pkg/src`` (the read-only upstream checkout, only in
     the build container).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
INSTALL_DIR = ROOT / "baseline" / "_ref"
UPSTREAM_SRC = Path("/root/reference/pkg/src")


def candidates():
    env = os.environ.get("ASTRAEA_REFERENCE")
    out = [Path(env)] if env else []
    return out + [INSTALL_DIR, UPSTREAM_SRC]


def load():
    """Return the ``agentsched`` module; raise ImportError loudly if absent."""
    try:
        import agentsched
        return agentsched
    except ImportError:
        pass
    for cand in candidates():
        if (cand / "agentsched" / "__init__.py").exists():
            if str(cand) not in sys.path:
                sys.path.insert(0, str(cand))
            import agentsched
            return agentsched
    raise ImportError(
        "the reference package 'agentsched' was not found (looked in: "
        + ", ".join(str(c) for c in candidates())
        + "); run __graft_entry__.build() to install it into baseline/_ref")


def install(force: bool = False) -> bool:
    """``pip install --no-index --target baseline/_ref`` of the upstream
    package (from a /tmp copy: /root/reference is read-only). Returns True
    when an install happened. No-op when the upstream checkout is absent
    (the GPU box, which receives the installed copy with the snapshot)."""
    import shutil
    import subprocess
    import tempfile
    if (INSTALL_DIR / "agentsched" / "__init__.py").exists() and not force:
        return False
    pkg = UPSTREAM_SRC.parent
    if not (pkg / "pyproject.toml").exists():
        return False
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(pkg, src)
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                        "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(INSTALL_DIR),
                        "--upgrade", str(src)], check=True, stdout=subprocess.DEVNULL)
    return True
