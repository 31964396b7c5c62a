"""NEXT-2 — parameter-offset discovery ("performs a byte-pattern match with the known
placeholder pointers within the buffer to identify the correct offsets").

find_param_offset(image, pattern): the unique offset of the 8-byte little-endian `pattern` on an
8-byte-aligned boundary of `image`; raises NotFound (no match) or Ambiguous (>= 2 matches).
A plain linear scan, pinned by the SPEC worked examples (offset 24 in a 40-byte image, absent ->
NotFound, matches at 8 and 32 -> Ambiguous) and randomized planted images.
"""
from __future__ import annotations

import struct


class NotFound(Exception):
    pass


class Ambiguous(Exception):
    pass


def find_param_offset(image: bytes, pattern: int) -> int:
    pat = struct.pack("<Q", pattern & 0xFFFFFFFFFFFFFFFF)
    hits = [off for off in range(0, len(image) - 7, 8) if image[off:off + 8] == pat]
    if not hits:
        raise NotFound()
    if len(hits) > 1:
        raise Ambiguous(hits)
    return hits[0]
