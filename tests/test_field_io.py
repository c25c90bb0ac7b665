"""UCVF / CSV / P5 I/O against bytes the reference wrote
(tests/golden/io.npz from critprob.field_io).  Host-side checks run on CPU;
the device streaming load and the device-side heatmap are marked gpu."""

import os

import numpy as np
import pytest

from paper_2407_18015_b200 import field_io as fio
from paper_2407_18015_b200.fields import EnsembleStack, ProbabilityField


def _prob(io):
    return ProbabilityField(io["prob/min"].copy(), io["prob/max"].copy(), io["prob/saddle"].copy(),
                            io["prob/valid"].copy())


def test_ensemble_ucvf_bytes_and_roundtrip(golden, tmp_path):
    io, fit = golden["io"], golden["fit"]
    stack = EnsembleStack(fit["ens/ackley"])
    p = tmp_path / "e.ucvf"
    fio.save_ensemble(stack, p)
    assert np.array_equal(np.frombuffer(p.read_bytes(), np.uint8), io["ensemble_ucvf"])
    back = fio.load_ensemble(p)
    assert np.array_equal(back.values, stack.values)


def test_probability_ucvf_and_csv_bytes(golden, tmp_path):
    io = golden["io"]
    prob = _prob(io)
    fio.save_probability_field(prob, tmp_path / "p.ucvf")
    assert np.array_equal(np.frombuffer((tmp_path / "p.ucvf").read_bytes(), np.uint8), io["prob_ucvf"])
    fio.save_probability_field(prob, tmp_path / "p.csv", format="csv")
    assert np.array_equal(np.frombuffer((tmp_path / "p.csv").read_bytes(), np.uint8), io["prob_csv"])
    back = fio.load_probability_field(tmp_path / "p.csv", format="csv")
    assert np.array_equal(back.p_min, prob.p_min) and np.array_equal(back.valid, prob.valid)
    back = fio.load_probability_field(tmp_path / "p.ucvf")
    assert np.array_equal(back.p_min, prob.p_min.astype(np.float32).astype(np.float64))


def test_ucvf_errors(tmp_path):
    bad = tmp_path / "bad.ucvf"
    bad.write_bytes(b"NOTUCVF 1 1 1\n" + b"\0" * 4)
    with pytest.raises(fio.UcvfFormatError):
        fio.load_ensemble(bad)
    bad.write_bytes(b"UCVF1 2 2 1\n" + b"\0" * 12)
    with pytest.raises(fio.UcvfPayloadError):
        fio.load_ensemble(bad)
    bad.write_bytes(b"UCVF1 1 1 1\n" + np.array([np.inf], "<f4").tobytes())
    with pytest.raises(fio.UcvfValueError):
        fio.load_ensemble(bad)
    bad.write_bytes(b"UCVF1 0 1 1\n")
    with pytest.raises(fio.UcvfFormatError):
        fio.load_ensemble(bad)
    assert issubclass(fio.UcvfValueError, fio.UcvfError)


def test_scalar_field_roundtrip(tmp_path):
    r = np.random.default_rng(1).uniform(0, 5, (6, 9))
    fio.save_scalar_field(r, tmp_path / "s.ucvf")
    back = fio.load_scalar_field(tmp_path / "s.ucvf")
    assert np.array_equal(back, r.astype(np.float32).astype(np.float64))
    with pytest.raises(ValueError):
        fio.save_scalar_field(np.ones(4), tmp_path / "x.ucvf")


@pytest.mark.gpu
def test_device_stream_load_and_heatmap(golden, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    io, fit = golden["io"], golden["fit"]
    p = tmp_path / "e.ucvf"
    p.write_bytes(io["ensemble_ucvf"].tobytes())
    st = fio.load_ensemble(p, device=True)
    assert st.on_device and np.array_equal(st.values.cpu().numpy(), fit["ens/ackley"])
    # chunked streaming path (tiny pinned chunks)
    w, h, dev = fio._read_device(p, chunk_bytes=1000)
    assert np.array_equal(dev.cpu().numpy(), fit["ens/ackley"])
    bad = tmp_path / "bad.ucvf"
    vals = fit["ens/ackley"].copy()
    vals[3, 4, 5] = np.nan
    bad.write_bytes(b"UCVF1 13 11 24\n" + vals.astype("<f4").tobytes())
    with pytest.raises(fio.UcvfValueError):
        fio.load_ensemble(bad, device=True)
    prob = _prob(io)
    for ch in ("min", "max", "saddle"):
        for g in (1.0, 0.5, 2.2):
            out = tmp_path / "h.pgm"
            fio.export_heatmap(prob, ch, out, gamma=g)
            assert np.array_equal(np.frombuffer(out.read_bytes(), np.uint8), io[f"heat/{ch}/{g}"]), (ch, g)
