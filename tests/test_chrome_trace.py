"""Chrome trace export of the device event trace (reference
write_chrome_trace, sim.cpp:597-610) on synthetic records: CTA lifetimes
become "X" spans per lane, tile events zero-length "X" events."""
import json

from paper_2406_06858_b200 import comm as CM


def _ev(event, rank, row, col, target, ns, lts):
    return {"event": event, "rank": rank, "tile_row": row, "tile_col": col, "target": target, "wall_ns": ns,
            "logical_ts": lts}


def test_chrome_trace_spans_and_events(tmp_path):
    events = [_ev("launch", 0, 3, 0, 0, 0, 1), _ev("compute_start", 0, 1, 2, 5, 1500, 2),
              _ev("signal_set", 0, 1, 0, 1, 1000, 3), _ev("launch", 0, 3, 1, 0, 9000, 4)]
    d = CM.chrome_trace(events)
    xs = d["traceEvents"]
    span = [x for x in xs if x["name"] == "cta 3"]
    assert span == [{"name": "cta 3", "ph": "X", "ts": 0.0, "dur": 9.0, "pid": 0, "tid": 3}]
    inst = [x for x in xs if x["tid"] == -1]
    assert {x["name"] for x in inst} == {"compute_start (1,2)", "signal_set (1,0)"}
    assert all(x["ph"] == "X" and x["dur"] == 0 for x in inst)
    p = tmp_path / "t.json"
    CM.write_chrome_trace(str(p), events)
    assert json.loads(p.read_text()) == d
