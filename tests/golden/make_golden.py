"""Writes tests/golden/edge_hash.json from the library routine sklearn.utils.murmurhash3_32
(Eq. 4, reading R4: LE32 u || LE32 v, seed 0, mod 2^31).  Calls no repo code."""
import json
import os
import struct

from sklearn.utils import murmurhash3_32

pairs = [[0, 1], [1, 0], [1, 2], [2, 1], [0, 0], [123456, 654321], [2147483646, 0], [16777215, 16777214]]
hs = [murmurhash3_32(struct.pack("<II", u, v), seed=0, positive=True) % (2**31) for u, v in pairs]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "edge_hash.json")
json.dump({"source": "sklearn.utils.murmurhash3_32 (MurmurHash3 x86_32) of LE32(u)||LE32(v), seed 0, mod 2^31; "
                     "Eq. 4 PAPER.md:222-225, reading R4; written by tests/golden/make_golden.py",
           "pairs": pairs, "hash": hs}, open(out, "w"), indent=1)
