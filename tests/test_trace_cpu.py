"""Trace feed (trace.py, mirrors hr/workloads/trace.py): exact dump/parse round
trips, the reference's format errors, and the BH force stream generated from
the oracle's lists equals the REFERENCE's recorded stream line for line
(tests/golden/trace_nbody3d_1500.txt, made by make_trace_golden.py)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2008_05712_b200 import trace
from paper_2008_05712_b200.errors import TraceFormatError


def _stream():
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    ps = gen.gen_particles(1500, 5, clustering=0.6, dim=3)
    t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    lists = orc.build_interaction_lists(t, 0.6)
    return trace.nbody_stream(lists.ptr, lists.ids, lists.item_count, seed=5)


def test_stream_equals_reference_golden():
    ref = trace.parse_trace(os.path.join(GOLDEN, "trace_nbody3d_1500.txt"))
    ours = _stream()
    assert len(ours) == len(ref)
    assert ours == ref  # arrival times (float bits), buffers, items, bytes


def test_roundtrip_exact(tmp_path):
    recs = _stream()[:50] + [trace.TraceRecord(0.1 + 0.2, "md", (3, 4), 12, 48)]
    assert trace.trace_roundtrip(recs, tmp_path / "t.txt") == []


@pytest.mark.parametrize("line,msg", [("1.0 force 1,2 3", "expected 5 fields"), ("x force 1 3 48", "could not"),
                                      ("1.0 force 1,2 0 48", "at least one item"), ("1.0 force 1,a 3 48", "")])
def test_format_errors(tmp_path, line, msg):
    p = tmp_path / "bad.txt"
    p.write_text("# header\n\n" + line + "\n")
    with pytest.raises(TraceFormatError) as e:
        trace.parse_trace(p)
    assert e.value.line_no == 3
    assert msg in str(e.value)
