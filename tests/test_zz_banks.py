"""The bank permutation of the B = 16 rank-ordered buffers (csrc/zz_banks.cuh, tools/gen_zz_banks.py):
a bijection inside each 32-rank row, one wavefront per D-fragment store slot, and 16 distinct
banks mod 16 per half row (the DD sweep's two-block test reads)."""
import os
import re
import sys

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "tools"))
import gen_zz_banks as g  # noqa: E402


def header_table():
    src = open(os.path.join(ROOT, "paper_2001_09632_b200", "csrc", "zz_banks.cuh")).read()
    body = src[src.index("kZzBank16[256] = {"):]
    vals = [int(v) for v in re.findall(r"\d+", body[body.index("{"):body.index("}")])]
    assert len(vals) == 256
    return vals


def test_header_matches_generator():
    assert header_table() == [v for row in g.bank_perm() for v in row]


def test_bank_properties():
    bank = header_table()
    slot = g.slot_of_rank()
    for row in range(8):
        assert sorted(bank[32 * row:32 * row + 32]) == list(range(32))
        for h in range(2):
            half = bank[32 * row + 16 * h:32 * row + 16 * h + 16]
            assert len({b % 16 for b in half}) == 16
    for s in range(8):
        banks = [bank[r] for r in range(256) if slot[r] == s]
        assert len(banks) == 32 and len(set(banks)) == 32
    # the slot map is the mma.sync D fragment of the transposed forward (mma_dct.cuh dslot_row/col)
    rank = g.zigzag_rank()
    assert rank[0] == 0 and rank[1] == 1 and rank[16] == 2 and rank[255] == 255
