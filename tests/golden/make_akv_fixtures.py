"""Generate the AKV1 format fixtures (acceptance 7).

Bytes are packed by hand from the format definition (not through
paper_2409_16546_b200.data_io), so the fixtures check the implementation
independently.  Run from the repo root: python tests/golden/make_akv_fixtures.py
"""
import os
import struct

import numpy as np

D = os.path.join(os.path.dirname(os.path.abspath(__file__)), "akv")
# +0, -0, min subnormal; 1.0, max finite, -inf
WORDS = np.array([[0x0000, 0x8000, 0x0001], [0x3C00, 0x7BFF, 0xFC00]], dtype="<u2")


def main():
    os.makedirs(D, exist_ok=True)
    hdr = b"AKV1" + bytes([1, 1, 0, 0]) + struct.pack("<I", 2) + struct.pack("<2I", 2, 3)
    good = hdr + WORDS.tobytes()
    assert len(good) == 32  # 20-byte header + 12-byte payload
    files = {
        "golden_2x3.akv": good,
        "bad_magic.akv": b"AKV2" + good[4:],
        "truncated.akv": good[:-3],
        "bad_dtype.akv": b"AKV1" + bytes([1, 2, 0, 0]) + good[8:],
    }
    for name, data in files.items():
        with open(os.path.join(D, name), "wb") as f:
            f.write(data)


if __name__ == "__main__":
    main()
