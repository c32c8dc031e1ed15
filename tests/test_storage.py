"""IFKC chunk-cache files (reference cache.py:103-199): byte compatibility
with files the reference wrote (golden), round trips, corruption handling."""

import numpy as np
import pytest
import torch

from paper_2603_05353_b200 import DataFormatError
from paper_2603_05353_b200.storage import load_cache, save_cache


def test_loads_reference_files_and_rewrites_identical_bytes(golden_small, tmp_path):
    for key in ("tiny_ifkc_f64", "tiny_ifkc_f32"):
        raw = golden_small[key].tobytes()
        src = tmp_path / f"{key}.ifkc"
        src.write_bytes(raw)
        ckv = load_cache(src, device="cpu")
        dst = tmp_path / f"{key}_re.ifkc"
        save_cache(ckv, dst)
        assert dst.read_bytes() == raw
    ckv = load_cache(tmp_path / "tiny_ifkc_f64.ifkc", device="cpu")
    np.testing.assert_array_equal(ckv.keys.numpy(), golden_small["tiny_chunk_keys"][1])
    np.testing.assert_array_equal(ckv.values.numpy(), golden_small["tiny_chunk_values"][1])
    assert ckv.chunk_id == "c1" and ckv.length == 8
    c32 = load_cache(tmp_path / "tiny_ifkc_f32.ifkc", device="cpu")
    assert c32.keys.dtype == torch.float32
    np.testing.assert_array_equal(c32.keys.numpy(), golden_small["tiny_ifkc_f32_keys"])


def test_bf16_round_trip(tmp_path, golden_small):
    src = tmp_path / "a.ifkc"
    src.write_bytes(golden_small["tiny_ifkc_f64"].tobytes())
    ckv = load_cache(src, device="cpu", dtype=torch.bfloat16)
    save_cache(ckv, tmp_path / "b.ifkc")
    back = load_cache(tmp_path / "b.ifkc", device="cpu")
    assert back.keys.dtype == torch.bfloat16
    assert torch.equal(back.keys, ckv.keys) and torch.equal(back.values, ckv.values)


@pytest.mark.parametrize("how", ["flip", "version", "magic", "truncate"])
def test_corruption_detected(tmp_path, golden_small, how):
    data = bytearray(golden_small["tiny_ifkc_f64"].tobytes())
    if how == "flip":
        data[len(data) // 2] ^= 0x01
    elif how == "version":
        data[4] = 0x7F
    elif how == "magic":
        data[:4] = b"JUNK"
    else:
        data = data[:-40]
    p = tmp_path / "c.ifkc"
    p.write_bytes(bytes(data))
    with pytest.raises(DataFormatError):
        load_cache(p, device="cpu")
