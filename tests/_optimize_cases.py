"""Shared iteration over tests/golden/optimize.npz (made by tests/golden/make_golden.py from the
reference's optimize.hpp)."""
import hashlib

import numpy as np

HAND = ("hand", "anti", "constbits", "const8")
SPEC = ("dup16", "dup32", "dup32_load", "uni24", "accept10", "dup100", "dup256", "dup1000")


def codes_for(g, name):
    """(codes[n, wpc] u64, bits) of a fixture case."""
    if name in HAND:
        return g[name + "_codes"], int(g[name + "_bits"][0])
    from paper_1307_2982_b200 import gen_uniform
    from paper_1307_2982_b200.cli import gen_duplicated_bits

    kind, n, bits, block, seed = (int(x) for x in g[name + "_spec"])
    if kind == 0:
        return gen_duplicated_bits(n, bits, block, seed).raw_words(), bits
    return gen_uniform(n, bits, seed).raw_words(), bits


def parts_for(g, name):
    return [(int(m), int(s)) for m, s in g[name + "_parts"]]


def corr_matches(g, name, corr):
    """Bitwise: the full matrix where stored, else its sha256."""
    if name + "_corr" in g:
        return np.array_equal(np.ascontiguousarray(corr, np.float64).view(np.uint64),
                              g[name + "_corr"].view(np.uint64))
    want = bytes(g[name + "_corr_sha256"]).hex()
    return hashlib.sha256(np.ascontiguousarray(corr, np.float64).tobytes()).hexdigest() == want


def subs_of(g, key_part, key_lens):
    pos, lens = g[key_part], g[key_lens]
    out, at = [], 0
    for L in lens:
        out.append([int(x) for x in pos[at:at + int(L)]])
        at += int(L)
    return out
