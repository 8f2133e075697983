"""Every `file:line` citation into the reference (/root/reference/proj) names
lines inside the cited file, and a citation right after a function name
overlaps that function's definition (tools/check_citations.py).  Skipped where
the reference tree is absent (the GPU box)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj"), reason="reference tree absent")
def test_reference_citations_resolve():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import check_citations
    failures, total = check_citations.check()
    assert total > 200
    assert not failures, "\n".join(failures)
