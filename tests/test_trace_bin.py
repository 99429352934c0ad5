"""Binary trace ingest: exact round trip, loud failures."""
import numpy as np
import pytest

from paper_2605_05899_b200.errors import ParseError, ValidationError
from paper_2605_05899_b200.trace import (
    TraceGenConfig, generate_trace, load_trace_bin, save_trace_bin, trace_digest,
)


@pytest.mark.parametrize("kw", [dict(n_visual=576, n_text=64, layers=8, experts=8, k=2, seed=0),
                                dict(n_visual=100, n_text=10, layers=4, experts=64, k=6, seed=3, decode_steps=5,
                                     shared_experts=2)])
@pytest.mark.parametrize("mmap", [False, True])
def test_round_trip_is_exact(tmp_path, kw, mmap):
    tr = generate_trace(TraceGenConfig(**kw))
    p = str(tmp_path / "t.vmm")
    save_trace_bin(tr, p)
    back = load_trace_bin(p, mmap=mmap)
    assert trace_digest(back) == trace_digest(tr)
    assert back == tr
    assert back.phase_marks == tr.phase_marks and back.shared_experts == tr.shared_experts


def test_malformed_files_raise(tmp_path):
    tr = generate_trace(TraceGenConfig(n_visual=50, n_text=5, layers=3, experts=8, k=2, seed=1))
    p = tmp_path / "t.vmm"
    save_trace_bin(tr, str(p))
    raw = p.read_bytes()
    (tmp_path / "bad_magic").write_bytes(b"NOTTRACE" + raw[8:])
    with pytest.raises(ParseError):
        load_trace_bin(str(tmp_path / "bad_magic"))
    (tmp_path / "short").write_bytes(raw[:-8])
    with pytest.raises(ParseError):
        load_trace_bin(str(tmp_path / "short"))
    # a duplicate expert inside one route violates the trace invariants (trace.py:375-382)
    bad = tr.route_experts.copy()
    bad[1, 3, 1] = bad[1, 3, 0]
    tr2 = type(tr)(tr.layers, tr.experts, tr.k, bad, tr.route_gates, tr.saliency, tr.modality, tr.embedding,
                   tr.cluster, tr.phase_marks, tr.shared_experts)
    save_trace_bin(tr2, str(tmp_path / "dup"))
    with pytest.raises(ValidationError):
        load_trace_bin(str(tmp_path / "dup"))
