"""Known-answer vectors for the device RNG's Philox4x32-10 (tests/test_rng.py).

Two independent sources:
* Random123's published philox4x32_10 known-answer vectors (kat_vectors:
  zero, all-ones and pi-digit counter/key) -- listed below;
* 256 random (counter, key) pairs evaluated by PyTorch's CPU Philox engine
  (torch/include/ATen/core/PhiloxRNGEngine.h, at::philox_engine, compiled
  here with g++), whose key is the seed and whose counter is (offset lo,
  offset hi, subsequence lo, subsequence hi).

The three Random123 vectors are also checked against the torch engine, so
the fixture is pinned by both.  Run in the build container:
    python tests/golden/make_philox_kat.py
"""
import os
import subprocess
import tempfile

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
RANDOM123 = [  # (ctr[4], key[2]) -> out[4]
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]
SRC = r"""
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdint>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    at::philox_engine e((uint64_t)k0 | ((uint64_t)k1 << 32), (uint64_t)c2 | ((uint64_t)c3 << 32), 0);
    e.set_offset((uint64_t)c0 | ((uint64_t)c1 << 32));
    unsigned a = e(), b = e(), c = e(), d = e();
    printf("%08x %08x %08x %08x\n", a, b, c, d);
  }
}
"""


def torch_philox(ctr, key):
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "p.cpp"), os.path.join(d, "p")
        open(src, "w").write(SRC)
        subprocess.run(["g++", "-std=c++17", "-O1", "-I", inc, src, "-o", exe], check=True)
        lines = "".join(f"{c[0]:x} {c[1]:x} {c[2]:x} {c[3]:x} {k[0]:x} {k[1]:x}\n" for c, k in zip(ctr, key))
        out = subprocess.run([exe], input=lines, capture_output=True, text=True, check=True).stdout.split()
    return np.array([int(x, 16) for x in out], np.uint32).reshape(-1, 4)


def main():
    rng = np.random.default_rng(123)
    ctr = np.concatenate([np.array([c for c, _, _ in RANDOM123], np.uint32),
                          rng.integers(0, 2**32, (256, 4), dtype=np.uint64).astype(np.uint32)])
    key = np.concatenate([np.array([k for _, k, _ in RANDOM123], np.uint32),
                          rng.integers(0, 2**32, (256, 2), dtype=np.uint64).astype(np.uint32)])
    out = torch_philox(ctr, key)
    want = np.array([o for _, _, o in RANDOM123], np.uint32)
    assert np.array_equal(out[:3], want), "torch's engine disagrees with Random123's vectors"
    np.savez_compressed(os.path.join(HERE, "philox_kat.npz"), ctr=ctr, key=key, out=out)
    print(f"wrote {len(ctr)} vectors")


if __name__ == "__main__":
    main()
