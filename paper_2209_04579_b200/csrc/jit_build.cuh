// Skeleton of a specialised build-side kernel, compiled at run time by NVRTC
// (jit.cu) after the generated hook
//
//   B_ROWS                                   rows per thread
//   void b_rows(s, r0, stride, pass, key, flags)
//        filter terms, string terms, LIKE flags and child probes of rows
//        r0 + j * stride (j < B_ROWS), straight-line with every constant
//        folded and every independent load issued first (fused.cu's generator)
//
//   B_ASSIGN, B_ZREC                          group-assigning build, words of
//                                            the group record zeroed per slot
//
// The rest is k_build's (fused_kernels.cuh): the group of a group-assigning
// build is its key slot (its state zeroed by the inserted row), the direct-
// address insert (plain stores; k_build_verify flags a key inserted twice, the
// 1:N join the fused contract excludes) and the presence bits OR-reduced per
// warp, a key inserted twice flagged from the bitmap words (presence_insert).
#pragma once

namespace tqp {
namespace fz {

extern "C" __global__ void __launch_bounds__(kThreads) q_build(const BuildSpec s) {
  unsigned dup = 0;
  const long long span = static_cast<long long>(blockDim.x) * B_ROWS;
  for (long long base0 = static_cast<long long>(blockIdx.x) * span; base0 < s.n;
       base0 += static_cast<long long>(gridDim.x) * span) {
    bool pass[B_ROWS];
    long long key[B_ROWS];
    unsigned flags[B_ROWS];
    b_rows(s, base0 + threadIdx.x, blockDim.x, pass, key, flags);
    unsigned old[B_ROWS], set[B_ROWS];
#pragma unroll
    for (int j = 0; j < B_ROWS; ++j) {
      old[j] = set[j] = 0u;
      if (!__any_sync(0xffffffffu, pass[j])) continue;  // warp-uniform: nothing to insert
      const long long r = base0 + j * blockDim.x + threadIdx.x;
      long long idx = -1;
      if (pass[j]) {
        idx = key[j] - s.kmin;
        if (idx < 0 || idx >= s.range) {
          atomicExch(reinterpret_cast<unsigned long long*>(s.err), 1ULL);
          idx = -1;
        } else {
#if B_ASSIGN
          {  // the group is the key slot: zero its record (whole sectors)
            ulonglong2* rec = reinterpret_cast<ulonglong2*>(s.zrec + idx * B_ZREC);
#pragma unroll
            for (int w = 0; w < B_ZREC / 2; ++w) rec[w] = make_ulonglong2(0ULL, 0ULL);
          }
#endif
#if B_ROWREC
          // the row is kept in the record's count word (bits 32-63), no table
          reinterpret_cast<unsigned long long*>(s.zrec)[idx * B_ZREC] = static_cast<unsigned long long>(r + 1) << 32;
#else
          s.table[idx] = static_cast<unsigned long long>(r + 1) | (static_cast<unsigned long long>(flags[j]) << 57);
#endif
        }
      }
#if B_UNIQUE
      presence_insert_unique(s.bitmap, idx);
#else
      presence_insert(s.bitmap, idx, old[j], set[j], dup);
#endif
    }
#pragma unroll
    for (int j = 0; j < B_ROWS; ++j) dup |= old[j] & set[j];
  }
  build_dup_check(dup, s.err);
}

}  // namespace fz
}  // namespace tqp
