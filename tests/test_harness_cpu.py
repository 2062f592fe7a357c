"""Host-side harness (no GPU): KVT1 tensor files, synthetic workloads, bench configs and the
CLI's shape-only verb (reference: sikv/harness/*, tests/test_tensorfile.py / test_cli.py)."""

import json

import numpy as np
import pytest

from paper_2603_14224_b200.harness import bench as bn
from paper_2603_14224_b200.harness.cli import main
from paper_2603_14224_b200.harness.synth import gen_synthetic
from paper_2603_14224_b200.harness.tensorfile import TensorFormatError, load_tensor, save_tensor
from paper_2603_14224_b200.synth import gen_unit


def test_tensorfile_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(0)
    p = tmp_path / "a.kvt"
    for shape in [(3,), (2, 5), (1, 2, 3)]:
        a = rng.standard_normal(shape).astype(np.float32)
        save_tensor(a, p)
        b = load_tensor(p)
        assert b.tobytes() == a.tobytes() and b.shape == a.shape and b.flags.writeable
    save_tensor(np.array([1.0, 2.5], dtype=np.float64), p, dtype="f16")
    np.testing.assert_array_equal(load_tensor(p), [1.0, 2.5])
    raw = p.read_bytes()
    for blob, msg in [(b"XXXX" + raw[4:], "magic"), (raw[:4] + b"\x02\x00" + raw[6:], "version"),
                      (raw[:6] + b"\x07" + raw[7:], "dtype code 7"), (raw[:5], "shorter than"),
                      (raw[:10], "truncated dims"), (raw + b"\x00\x00", "6 bytes, expected 4")]:
        p.write_bytes(blob)
        with pytest.raises(TensorFormatError, match=msg):
            load_tensor(p)
    with pytest.raises(ValueError, match="dtype"):
        save_tensor(np.ones(2), p, dtype="f64")


def test_gen_synthetic_is_the_unit_generator():
    w = gen_synthetic(300, 16, 5, seed=4, window=7)
    u = gen_unit(300, 16, 5, 4, window=7, bf16=False)
    for a, b in [(w.keys, u.keys), (w.values, u.values), (w.queries, u.queries), (w.window, u.window),
                 (w.paired_rows, u.paired)]:
        np.testing.assert_array_equal(a, b)
    assert (w.tokens, w.dim) == (300, 16)
    with pytest.raises(ValueError, match="correlated_fraction"):
        gen_synthetic(10, 4, 1, 0, correlated_fraction=1.5)


def test_bench_config_contract():
    with pytest.raises(ValueError, match="exactly one"):
        bn.BenchConfig()
    with pytest.raises(ValueError, match="ablation"):
        bn.BenchConfig(budget=3, ablation="nope")
    assert bn.BenchConfig(sparsity=0.075, tokens=4096).target_tokens == 307
    rec = bn.make_record("memory", bn.BenchConfig(budget=0), bits_per_token=896)
    assert set(rec) == set(bn.RECORD_KEYS)


def test_cli_memory_verb(capsys, tmp_path):
    out = tmp_path / "r.jsonl"
    assert main(["memory", "--tokens", "4096", "--check", "--out", str(out)]) == 0
    rec = json.loads(capsys.readouterr().out.strip())
    assert (rec["bench"], rec["bits_per_token"], rec["savings_fraction"]) == ("memory", 896, 0.78125)
    assert json.loads(out.read_text())["bench"] == "memory"
    with pytest.raises(SystemExit):
        main(["frobnicate"])
