"""Every device sorter once on small, awkward shapes (tools/sanitize_probe.py),
checked against numpy / the oracle.  The same probe is the workload of the
CHECKED build (device-side bounds checks; profiles/round2/sanitizer.md)."""

import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu


def test_sanitize_probe():
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import sanitize_probe
    sanitize_probe.main()
