"""Import the live reference package ``pxst`` (TEST INFRASTRUCTURE ONLY).

Works only where ``/root/reference`` exists (the build container), never on
the GPU box.  ``pxst/__init__.py:10`` imports ``cxi_io`` which needs h5py
(``cxi_io.py:18``); h5py is not installed and the hot path never touches it,
so an empty stub module is registered first.  Used to pin the oracle
(``tests/test_oracle_golden.py``) and to write golden vectors
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import os
import sys
import types

REF_SRC = os.environ.get("PXST_REFERENCE_SRC", "/root/reference/pkg/src")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "pxst"))


def load():
    """Return the reference ``pxst`` package (raises ImportError if absent)."""
    if not available():
        raise ImportError(f"reference sources not found at {REF_SRC}")
    if "h5py" not in sys.modules:
        sys.modules["h5py"] = types.ModuleType("h5py")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import pxst  # noqa: E402
    return pxst
