"""Plan wire format (codegen.py:619-798) restated without the reference package."""

import shutil

import numpy as np
import pytest

from conftest import GOLDEN, bits
from paper_2110_12865_b200.plan import load_plan, save_plan, slot_addresses


def test_save_is_byte_identical_to_reference(golden, tmp_path):
    # manifest.json + data.blob written by the reference's save_plan
    save_plan(golden.plan, tmp_path)
    assert (tmp_path / "manifest.json").read_bytes() == (golden.dir / "manifest.json").read_bytes()
    assert (tmp_path / "data.blob").read_bytes() == (golden.dir / "data.blob").read_bytes()


def test_round_trip_keeps_addresses(golden, tmp_path):
    save_plan(golden.plan, tmp_path)
    again = load_plan(tmp_path)
    for ka, kb in zip(golden.plan.kernels, again.kernels):
        for a, b in zip(slot_addresses(golden.plan, ka), slot_addresses(again, kb)):
            assert np.array_equal(a, b)


def _copy(name, tmp_path):
    dst = tmp_path / name
    shutil.copytree(GOLDEN / name, dst)
    return dst


def test_corrupt_magic_rejected(tmp_path):
    d = _copy("toy256", tmp_path)
    blob = bytearray((d / "data.blob").read_bytes())
    blob[0] = 0x58
    (d / "data.blob").write_bytes(bytes(blob))
    with pytest.raises(ValueError):
        load_plan(d)


def test_truncated_blob_rejected(tmp_path):
    d = _copy("toy256", tmp_path)
    raw = (d / "data.blob").read_bytes()
    (d / "data.blob").write_bytes(raw[: len(raw) // 2])
    with pytest.raises(ValueError):
        load_plan(d)


def test_bad_version_rejected(tmp_path):
    d = _copy("toy256", tmp_path)
    blob = bytearray((d / "data.blob").read_bytes())
    blob[4] = 2
    (d / "data.blob").write_bytes(bytes(blob))
    with pytest.raises(ValueError):
        load_plan(d)


def test_position_out_of_range_rejected(tmp_path):
    d = _copy("spgemm_n60_k4", tmp_path)
    raw = bytearray((d / "data.blob").read_bytes())
    raw[8 + 12: 8 + 12 + 4] = (0xFFFFFFF0).to_bytes(4, "little")
    (d / "data.blob").write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        load_plan(d)


def test_unsupported_manifest_format(tmp_path):
    d = _copy("toy256", tmp_path)
    m = (d / "manifest.json").read_text().replace('"format":1', '"format":2')
    (d / "manifest.json").write_text(m)
    with pytest.raises(ValueError):
        load_plan(d)
