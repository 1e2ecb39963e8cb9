"""CPU checks of the parity helpers (tests/parity.py) themselves: on outputs produced by the oracle
they pass, and a single corrupted entry in any instance -- sampled or not -- fails them (the
sampled mode catches it through the eigen-checksum when the entry is not sampled)."""
import numpy as np
import pytest

import oracle
import parity
import synth


@pytest.mark.parametrize("p", [synth.P998, synth.GOLDILOCKS])
@pytest.mark.parametrize("full", [True, False])
def test_check_matvec_passes_and_catches(p, full, monkeypatch, tmp_path):
    monkeypatch.setenv("FCIRC_PARITY_LOG", str(tmp_path / "log.jsonl"))
    inp = synth.matvec_inputs(p, 64, 5, seed=9)
    c = np.stack([oracle.fcirc_entries(p, inp["f"], inp["a"][k], inp["b"][k]) for k in range(5)])
    rec = parity.check_matvec("t", inp, c, full=full, sample=8)
    assert rec["instances"] == 5 and rec["mismatches"] == 0
    assert rec["entries"] == (5 * 64 if full else 5 * (8 + 6))
    bad = c.copy()
    bad[3, 40] = (int(bad[3, 40]) + 1) % p
    with pytest.raises(AssertionError):
        parity.check_matvec("t", inp, bad, full=full, sample=8)
    assert (tmp_path / "log.jsonl").read_text().count("\n") == 2


def test_check_matvec_f_minus_one_and_one(monkeypatch, tmp_path):
    monkeypatch.setenv("FCIRC_PARITY_LOG", str(tmp_path / "log.jsonl"))
    for mode in ("one", "minus_one"):
        inp = synth.matvec_inputs(synth.P998, 32, 3, seed=4, f_mode=mode)
        c = np.stack([oracle.fcirc_entries(inp["p"], inp["f"], inp["a"][k], inp["b"][k]) for k in range(3)])
        parity.check_matvec(mode, inp, c, full=False, sample=4)
        c[1, 7] ^= 1
        with pytest.raises(AssertionError):
            parity.check_matvec(mode, inp, c, full=False, sample=0)   # checksum alone catches it


def test_check_polymul(monkeypatch, tmp_path):
    monkeypatch.setenv("FCIRC_PARITY_LOG", str(tmp_path / "log.jsonl"))
    inp = synth.polymul_inputs(synth.P998, 40, 30, 3, seed=2)
    c = np.stack([oracle.polymul_coeffs(synth.P998, inp["a"][k], inp["b"][k]) for k in range(3)])
    parity.check_polymul("t", inp, c)
    c[2, 50] = (int(c[2, 50]) + 5) % synth.P998
    with pytest.raises(AssertionError):
        parity.check_polymul("t", inp, c)
