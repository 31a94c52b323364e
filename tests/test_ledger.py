"""The logical exchange ledger in the reference's schema (CommLedger,
simgroup.py:54-172) and the zero-tolerance ledger law of verify.check_ledger
(verify.py:146-169) for the Ulysses scheme -- host logic, no GPU."""

import csv
import io

from paper_2309_14509_b200.comm import CommLedger, CommRecord, check_ledger
from oracle import ulysses_oracle as O


def ulysses_ledger(n, b, d, p, layers=1, backward=False):
    """What one rank records: per layer 4 flips of a local n/P*b*d tensor
    (ulysses.py:144-155), mirrored by the backward (ulysses.py:213-226)."""
    led = CommLedger()
    local = n // p * b * d
    agg, eg = O.all_to_all_metering(local, p)
    labels = ["attn.q.seq2head", "attn.k.seq2head", "attn.v.seq2head", "attn.ctx.head2seq"]
    if backward:
        labels += ["bwd.ctx.seq2head", "bwd.q.head2seq", "bwd.k.head2seq", "bwd.v.head2seq"]
    for _ in range(layers):
        for lab in labels:
            led.append(CommRecord("all_to_all", lab, agg, eg))
    return led


def test_ledger_law_holds_and_matches_costmodel():
    for n, b, d, p, layers, bwd in [(64, 1, 32, 4, 1, False), (128, 2, 64, 8, 2, True), (16, 1, 8, 1, 1, False)]:
        led = ulysses_ledger(n, b, d, p, layers, bwd)
        ok, measured, predicted = check_ledger(led, n, b, d, p, layers, bwd)
        assert ok and measured == predicted
        assert predicted == O.ulysses_volume(n, b, d, p) * layers * (2 if bwd else 1)


def test_ledger_law_catches_a_missing_or_wrong_record():
    led = ulysses_ledger(64, 1, 32, 4)
    assert not check_ledger(CommLedger(led[:3]), 64, 1, 32, 4)[0]
    bad = CommLedger(led[:3] + [CommRecord("all_to_all", "x", 64 * 32, 1)])
    assert not check_ledger(bad, 64, 1, 32, 4)[0]


def test_csv_and_json_in_reference_schema():
    led = ulysses_ledger(64, 1, 32, 4)
    rows = list(csv.reader(io.StringIO(led.to_csv_text())))
    assert rows[0] == ["step_label", "collective", "aggregate_elements", "per_rank_egress_elements"]
    assert rows[1] == ["attn.q.seq2head", "all_to_all", str(64 * 32), str(64 * 32 // 4 // 4 * 3)]
    assert led.to_json_obj()[3]["step_label"] == "attn.ctx.head2seq"
    assert led.counts_by_collective() == {"all_to_all": 4}
    assert led.total_egress("all_to_all", "attn.q.seq2head") == 64 * 32 // 16 * 3
