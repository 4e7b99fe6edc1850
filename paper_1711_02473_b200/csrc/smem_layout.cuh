// Compile-time shared-memory padding search.
//
// fp64 shared accesses: a warp's 32 lanes x 8 B are served in two 16-lane
// phases; within a phase, lanes whose 8-byte words fall in the same bank
// (word index mod 16) but at different addresses serialise.  For the line
// kernels every stage has the shape
//     address(lane, k) = base(lane) + k * stride      (k = loop index)
// so the conflict degree depends only on {base(lane) mod 16}.  The helpers
// below evaluate that degree for an affine 3D layout and pick the padding
// that minimises the worst stage.
#pragma once

namespace sfk {

// Worst conflict degree over the two half-warps for lane addresses base[0..31].
__host__ __device__ constexpr int conflict_degree(const int* base, int nlanes) {
  int worst = 1;
  for (int h = 0; h < 2; ++h) {
    for (int b = 0; b < 16; ++b) {
      int distinct = 0;
      for (int l = h * 16; l < h * 16 + 16 && l < nlanes; ++l) {
        if (((base[l] % 16) + 16) % 16 != b) continue;
        bool seen = false;
        for (int k = h * 16; k < l; ++k)
          if (base[k] == base[l]) seen = true;
        if (!seen) ++distinct;
      }
      if (distinct > worst) worst = distinct;
    }
  }
  return worst;
}

// Lanes enumerate (cell, a, b) with b fastest (extents ea, eb); the address
// of lane (c, a, b) is c*cs + a*sa + b*sb.  Returns the worst degree over
// the first warp (later warps see the same pattern shifted by whole cells or
// rows, which is checked by also scanning a warp that starts mid-cell).
__host__ __device__ constexpr int pattern_degree(int ea, int eb, int sa, int sb, int cs,
                                                 int cells) {
  int worst = 1;
  const int per = ea * eb;
  const int total = per * cells;
  for (int start = 0; start < total; start += 32) {
    int base[32] = {};
    int n = 0;
    for (int l = 0; l < 32 && start + l < total; ++l) {
      const int t = start + l;
      const int c = t / per, r = t % per;
      const int a = r / eb, b = r % eb;
      base[n++] = c * cs + a * sa + b * sb;
    }
    const int d = conflict_degree(base, n);
    if (d > worst) worst = d;
  }
  return worst;
}

}  // namespace sfk
