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
    save_cache(ckv, tmp_path / "b.ifkc", precision="bf16")  # the compact native file (code 2)
    back = load_cache(tmp_path / "b.ifkc", device="cpu")
    assert back.keys.dtype == torch.bfloat16
    assert torch.equal(back.keys, ckv.keys) and torch.equal(back.values, ckv.values)
    # default: a bf16 cache is written as exact f32 (code 0), which the reference can read
    save_cache(ckv, tmp_path / "c.ifkc")
    raw = (tmp_path / "c.ifkc").read_bytes()
    n_id = int.from_bytes(raw[16:20], "little")
    assert raw[20 + n_id + 16 + 1] == 0  # precision code byte
    f32 = load_cache(tmp_path / "c.ifkc", device="cpu")
    assert f32.keys.dtype == torch.float32 and torch.equal(f32.keys, ckv.keys.float())


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


@pytest.mark.gpu
def test_reference_files_load_into_hbm(golden_small, tmp_path, cuda):
    """IFKC files the reference wrote (f64 and f32) straight into HBM, as
    stored and converted on the device (f32, bf16), via one pinned read."""
    paths = []
    for key in ("tiny_ifkc_f64", "tiny_ifkc_f32"):
        paths.append(tmp_path / f"{key}.ifkc")
        paths[-1].write_bytes(golden_small[key].tobytes())
    f64 = load_cache(paths[0], device="cuda")
    assert f64.keys.is_cuda and f64.keys.dtype == torch.float64
    np.testing.assert_array_equal(f64.keys.cpu().numpy(), golden_small["tiny_chunk_keys"][1])
    np.testing.assert_array_equal(f64.values.cpu().numpy(), golden_small["tiny_chunk_values"][1])
    as32 = load_cache(paths[0], device="cuda", dtype=torch.float32)
    np.testing.assert_array_equal(as32.keys.cpu().numpy(), golden_small["tiny_chunk_keys"][1].astype(np.float32))
    as16 = load_cache(paths[0], device="cuda", dtype=torch.bfloat16)
    assert torch.equal(as16.keys, f64.keys.to(torch.bfloat16))
    from paper_2603_05353_b200.storage import load_caches

    both = load_caches(paths, device="cuda", dtype=torch.float32)
    np.testing.assert_array_equal(both[1].keys.cpu().numpy(), golden_small["tiny_ifkc_f32_keys"])
    assert both[0].chunk_id == "c1" and both[0].length == 8
    # a device bf16 cache written by default as f32 reloads bit-identically
    save_cache(as16, tmp_path / "back.ifkc")
    back = load_cache(tmp_path / "back.ifkc", device="cuda", dtype=torch.bfloat16)
    assert torch.equal(back.keys, as16.keys) and torch.equal(back.values, as16.values)
