"""Host logic of the device async trace audit on synthetic
records: a valid publish order passes; reading a version that was not yet
published and a remembered reading that is not the previous fresh one are
both caught. Runs without a GPU."""
import numpy as np

import paper_2110_10762_b200 as pb


def rec(i, vf, vr, fonly=0, delta=0.5, t0=0, t1=10, cl=0):
    d = np.array([delta], dtype=np.float64).view(np.int64)[0]
    return [i, vf, vr, fonly, d, t0, t1, cl]


def valid_records():
    # p = 3: slice 1 reads slice 0 (always version 0)
    return np.array([
        rec(1, 0, 0, 0, t0=0, t1=10, cl=0),
        rec(2, 1, 0, 0, t0=5, t1=15, cl=1),   # overlaps the first: 2 in flight
        rec(3, 0, 0, 0, t0=6, t1=16, cl=2),   # stale read (slice 2 had 0 publishes at its read) is legal
        rec(3, 1, 0, 0, t0=20, t1=30, cl=0),  # remembered = previous fresh read (0)
        rec(2, 1, 1, 1, t0=21, t1=31, cl=1),
        rec(3, 2, 1, 0, t0=40, t1=50, cl=2),
        rec(3, 2, 2, 1, t0=60, t1=70, cl=0),
    ], dtype=np.int64)


def test_valid_trace_passes():
    r = valid_records()
    counts = np.array([0, 1, 2, 4])
    a = pb.audit_device_trace(r, 3, counts)
    assert a["ok"], a
    assert a["events"] == 7
    assert a["peak_in_flight"] == 3
    assert a["clusters_used"] == 3
    assert a["max_staleness"] == 1  # slice 3 read version 0 while slice 2 had published 1


def test_causality_violation_detected():
    r = valid_records()
    r[1, 1] = 2  # slice 2 claims version 2 of slice 1, which only ever published once
    a = pb.audit_device_trace(r, 3, np.array([0, 1, 2, 4]))
    assert not a["ok"] and a["causality_violations"] == 1


def test_provenance_violation_detected():
    r = valid_records()
    r[3, 2] = 1  # remembered version 1, but the previous fresh read of slice 3 was 0
    a = pb.audit_device_trace(r, 3, np.array([0, 1, 2, 4]))
    assert not a["ok"] and a["provenance_violations"] == 1


def test_count_mismatch_detected():
    a = pb.audit_device_trace(valid_records(), 3, np.array([0, 1, 2, 3]))
    assert not a["ok"] and a["counts_match"] is False


def test_trace_export_matches_reference_types():
    from paper_2110_10762_b200.async_parareal import device_records_to_trace
    tr = device_records_to_trace(valid_records(), 3, np.array([0, 1, 2, 4]), None, "converged")
    assert [e.component for e in tr.events] == [1, 2, 3, 3, 2, 3, 3]
    assert tr.events[1].reads == ((1, pb.FRESH_SLOT, 1), (1, pb.REMEMBERED_SLOT, 0))
    assert tr.events[0].delta == 0.5
    lines = tr.to_jsonl().strip().split("\n")
    assert len(lines) == 7
