// Shared-memory bank of each B = 16 zigzag rank inside its 32-rank row (tools/gen_zz_banks.py):
// rank r of a rank-ordered buffer lives at (r & ~31) | kZzBank16[r], so each mma.sync D-fragment
// store slot hits 32 distinct banks, 32-aligned runs stay conflict-free, and each half row hits
// 16 distinct banks mod 16 (two blocks' buffers 16 banks apart are read in one wavefront).
#pragma once
#include "common.cuh"
namespace abcs_b200 {
ABCS_DEV_TABLE unsigned char kZzBank16[256] = {
    1, 0, 3, 4, 2, 5, 9, 6, 7, 8, 10, 15, 11, 12, 13, 14, 17, 18, 16, 19, 20, 24, 21, 22, 23, 30, 25, 26, 31, 27, 28, 29,
    16, 10, 2, 4, 17, 13, 21, 7, 25, 14, 12, 11, 19, 6, 8, 15, 0, 3, 1, 20, 24, 5, 18, 22, 23, 9, 26, 27, 28, 29, 31, 30,
    1, 0, 18, 3, 21, 7, 6, 9, 8, 30, 10, 11, 13, 4, 12, 15, 16, 2, 19, 5, 23, 22, 17, 20, 25, 24, 26, 28, 27, 29, 14, 31,
    0, 17, 18, 20, 3, 21, 6, 23, 8, 25, 26, 11, 28, 29, 30, 15, 19, 16, 2, 1, 5, 22, 4, 7, 24, 9, 10, 12, 27, 13, 14, 31,
    0, 17, 2, 19, 4, 5, 6, 9, 7, 24, 27, 26, 29, 14, 31, 28, 18, 20, 16, 3, 22, 23, 21, 8, 10, 12, 25, 11, 15, 1, 13, 30,
    0, 18, 1, 3, 22, 21, 7, 25, 8, 12, 20, 26, 11, 29, 15, 30, 2, 19, 5, 17, 4, 6, 23, 24, 9, 16, 27, 10, 28, 13, 14, 31,
    16, 5, 17, 2, 4, 8, 23, 9, 26, 13, 28, 3, 27, 15, 6, 14, 18, 1, 20, 24, 0, 19, 21, 22, 25, 7, 10, 11, 29, 31, 12, 30,
    17, 20, 16, 2, 5, 19, 8, 6, 9, 26, 11, 7, 12, 30, 29, 31, 0, 1, 18, 3, 4, 21, 22, 23, 24, 25, 10, 27, 28, 13, 14, 15,
};
}  // namespace abcs_b200
