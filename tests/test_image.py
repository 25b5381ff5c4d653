"""FilterImage v1 on device (persist.hpp:14-66): serialize/deserialize/save/load
with the CRC-32 computed on the GPU, checked against the oracle's byte-serial
image and the reference's golden CRCs and error codes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2101_01719_b200 import SplitBlockFilter  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402
from paper_2101_01719_b200.filter import PersistError  # noqa: E402


def dev(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(cuda)


@pytest.mark.parametrize("nb", [1, 2, 3, 7, 255, 256, 2048, 2049, 4096, 65537, 1 << 20, 9_470_000 + 2049])
@pytest.mark.parametrize("hasher_id", [0, 1])
def test_image_matches_oracle(cuda, oracle, nb, hasher_id):
    rng = np.random.default_rng(nb)
    hs = rng.integers(0, 2**64, size=min(20 * nb, 3_000_000), dtype=np.uint64)
    f = SplitBlockFilter(nb, hasher_id=hasher_id)
    f.add_hashes(dev(hs, cuda))
    want = oracle.serialize(oracle.build(nb, hs), hasher_id)
    assert f.image_crc() == int.from_bytes(want[-4:], "little")
    img = f.serialize()
    assert img == want
    g = SplitBlockFilter.deserialize(img)
    assert g == f and g.hasher_id() == hasher_id and g.num_buckets() == nb


def test_golden_images(cuda, oracle, golden_units):
    for c in golden_units["filters"]:
        draws = oracle.mt19937_64(c["seed"], c["adds"])
        f = SplitBlockFilter(c["buckets"])
        f.add_hashes(dev(draws, cuda))
        assert f.image_crc() == c["image_crc"], c["name"]
        if "image_hex" in c:
            assert f.serialize().hex() == c["image_hex"]


def test_config3_image_crc_on_device(cuda, golden_configs):
    cfg = W.CONFIGS[3]
    st = W.StreamHandle(cfg.inserts)
    f = SplitBlockFilter(cfg.num_buckets)
    f.add_hashes(W.gen_inserts(st, 0, cfg.inserts.n))
    assert f.image_crc() == golden_configs["3"]["image_crc"]   # 128 MiB of blocks, 2048 segments


def test_deserialize_errors_match_reference_codes(cuda, oracle):
    f = SplitBlockFilter(3)
    f.add_hashes(dev([1, 2, 3], cuda))
    img = bytearray(f.serialize())
    cases = {
        "short": bytes(img[:20]),
        "long": bytes(img) + b"\0",
        "magic": bytes(b"X" + img[1:]),
        "version": bytes(img[:4] + b"\x02" + img[5:]),
        "crc_trailer": bytes(img[:-1] + bytes([img[-1] ^ 1])),
        "crc_payload": bytes(img[:30] + bytes([img[30] ^ 0x10]) + img[31:]),
    }
    zero = bytearray(oracle.serialize(oracle.new_blocks(1)))
    zero[9:17] = b"\0" * 8
    cases["zero_buckets"] = bytes(zero)
    for name, data in cases.items():
        want = oracle.deserialize(data)[0]
        assert want != 0, name
        with pytest.raises(PersistError) as ei:
            SplitBlockFilter.deserialize(data)
        assert ei.value.errc == want, name


def test_save_and_load(cuda, tmp_path):
    f = SplitBlockFilter(1000, hasher_id=1)
    f.add_hashes(dev(np.arange(1, 5001, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15), cuda))
    p = tmp_path / "f.sbbf"
    f.save(str(p))
    g = SplitBlockFilter.load(str(p))
    assert g == f and g.hasher_id() == 1
    with pytest.raises(PersistError) as ei:
        SplitBlockFilter.load(str(tmp_path / "missing.sbbf"))
    assert ei.value.code == "kIo"
