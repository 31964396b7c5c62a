"""NEXT-2 parameter-offset discovery: oracle pins (criterion 8 S:L561) and the
C-ABI host function against the oracle (no GPU needed)."""
import random
import struct

import pytest

from oracle import offsets as ooff


def test_spec_examples():
    pat = 0x00007F1234567890
    img = bytearray(40)
    img[24:32] = struct.pack("<Q", pat)
    assert ooff.find_param_offset(bytes(img), pat) == 24
    with pytest.raises(ooff.NotFound):
        ooff.find_param_offset(bytes(40), pat)
    img2 = bytearray(40)
    img2[8:16] = img2[32:40] = struct.pack("<Q", pat)
    with pytest.raises(ooff.Ambiguous):
        ooff.find_param_offset(bytes(img2), pat)


def test_unaligned_occurrence_is_ignored():
    pat = 0x1122334455667788
    img = bytearray(48)
    img[4:12] = struct.pack("<Q", pat)                                  # straddles a slot boundary
    with pytest.raises(ooff.NotFound):
        ooff.find_param_offset(bytes(img), pat)


def _randomized(rnd, n):
    size = 8 * rnd.randint(1, 64)
    img = bytearray(rnd.getrandbits(8) for _ in range(size))
    pat = rnd.getrandbits(64) | (1 << 47)
    slots = list(range(0, size, 8))
    k = rnd.choice([0, 1, 1, 1, 2])
    for off in rnd.sample(slots, min(k, len(slots))):
        img[off:off + 8] = struct.pack("<Q", pat)
    return bytes(img), pat


def test_randomized_1000_images_oracle_and_abi_agree():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx
    rnd = random.Random(8)
    for i in range(1000):                                               # S:L561 criterion 8
        img, pat = _randomized(rnd, i)
        try:
            ref = ("ok", ooff.find_param_offset(img, pat))
        except ooff.NotFound:
            ref = ("nf", None)
        except ooff.Ambiguous:
            ref = ("amb", None)
        try:
            got = ("ok", cgx.find_param_offset(img, pat))
        except cgx.CgxError as e:
            got = ({cgx.E_OFFSET_NOT_FOUND: "nf", cgx.E_OFFSET_AMBIGUOUS: "amb"}[e.status], None)
        assert got == ref, i
