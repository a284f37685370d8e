// Shared layouts and device helpers of the fused fact-scan pipelines.
// Compiled twice: into libtqp_b200.so (fused_kernels.cuh) and, embedded as a
// string, into every specialised pipeline kernel NVRTC builds at run time
// (jit.cu), so the host-filled TileSpec and both kernels share one layout.
// Self-contained: no CUDA runtime or C++ library headers.
#pragma once

#include <stdint.h>

#include "tqp_b200.h"

namespace tqp {
namespace fz {

constexpr int kMaxTerms = 8;
constexpr int kMaxProbes = 3;
constexpr int kMaxAcc = 8;
constexpr int kMaxFactors = 4;
constexpr int kMaxKeys = 4;
constexpr int kMaxStrTerms = 4;
constexpr int kMaxFlags = 7;
constexpr int kGroups = 8;  // MODE_SMALL per-CTA slot capacity (register accumulators)
constexpr int kGroupBits = 3;
constexpr int kMaxAccSmall = 6;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

enum OperandType : int { OT_I64 = 0, OT_F64 = 1, OT_U8 = 2 };
enum TermKind : int { TK_INT = 0, TK_F64 = 1, TK_TRUE = 2, TK_FALSE = 3 };
enum FactorKind : int { FK_X = 0, FK_K_MINUS_X, FK_K_PLUS_X, FK_X_MINUS_K, FK_X_PLUS_K, FK_X_TIMES_K, FK_CONST };
enum Mode : int { MODE_SCALAR = 0, MODE_SMALL = 1, MODE_BUILDGRP = 2, MODE_HASH = 3 };

// err[3]: why a fused unit handed its steps to the exact per-instruction path
// (err[0] != 0). Diagnostic only (TQP_DEBUG_FALLBACK prints it); the exact
// path then produces the reference's result or error.
enum FallbackReason : long long {
  FR_BUILD_RANGE = 11,     // build key outside the direct-address range
  FR_DUP_KEY = 12,         // a build key inserted twice (1:N join)
  FR_Q64_CONVERT = 13,     // an fp64 group value not exactly representable in Q64.64
  FR_Q64_RANGE = 14,       // max|value| x rows may reach 2^62: a Q64.64 group sum could wrap
  FR_LIMB_ROWS = 15,       // a group has >= kLimbMaxRows rows (limb words could overflow)
  FR_TOPK_BLOCK = 16,      // top-k: a block's candidate log overflowed
  FR_TOPK_FINAL = 17,      // top-k: too many final candidates (ties)
  FR_GROUP_VALUE = 18,     // a group output (AVG / epilogue) left the exact form
  FR_INT_RANGE = 19,       // int64 sum may overflow (|v| x rows >= 2^63)
  FR_HASH_FULL = 22,       // hash group / join table probe sequence exhausted
  FR_KEY_RANGE = 23,       // a group key digit outside its range (stale key range)
  FR_LIMB2 = 24,           // a value too wide for the 2-limb group sums (re-run with 3 limbs)
};

// A per-row operand: fact column (src = -1) or a column of the build-side
// root row matched by probe `src`.
struct Operand {
  const void* ptr = nullptr;
  int type = OT_I64;
  int src = -1;
  int col = -1;  // fact operands: column index in the staged tile
};

struct Term {
  Operand x;
  int kind = TK_TRUE;
  int op = TQP_EQ;
  long long ik = 0;
  double fk = 0.0;
};

// string predicate over STR8 rows: compare with a literal (zero-extended, as
// string_compare_rows, executor.cpp:72-108) or LIKE (substring_match,
// kernels.cpp:692-728)
struct StrTerm {
  const uint8_t* ptr = nullptr;
  int width = 1;
  int is_like = 0;
  int op = TQP_EQ;      // compare op when !is_like
  int anchor = TQP_START;
  int litlen = 0;
  unsigned char lit[48];
};

// factor = fa + fb * x, evaluated branch-free (fa/fb derived from `kind`):
// K - x == K + (-1)x and 1 * x == x exactly; padding factors are 1 + 0 * 0
struct Factor {
  Operand x;
  int kind = FK_X;
  double k = 0.0;
  double fa = 1.0, fb = 0.0;
};
constexpr int kFixedFactors = 3;

struct Acc {
  int is_int = 0;
  int base = -1;  // earlier accumulator whose factor product is this one's prefix
  int nf = 0;
  Factor f[kMaxFactors];
  int gate_probe = -1;  // value counts only if flag bit of probe is set
  int gate_bit = 0;
  double gate_else = 0.0;
};

// dense direct-address build table: entry 0 = empty, else
//   bits 0-31 rowid+1 | bits 57-63 flags; the group of a group-assigning
//   build is the key slot (key - kmin), valid where the presence bit is set
// A build whose key range is too wide for direct addressing is an
// open-addressing table instead (hkeys != nullptr): slot = hash(key) with
// linear probing at load <= 1/2, hkeys[slot] the key (kmin - 1 marks an
// empty slot: no key of the column is below kmin), table[slot] the entry.
// A build whose keys repeat (a 1:N join) is re-run with mult != nullptr:
// mult[slot] = the summed weight of the build rows with that key (a row's
// weight is the product of its own child probes' multiplicities); the fact
// scan then counts a row mult times and adds its values times mult.
struct Probe {
  Operand key;
  long long kmin = 0;
  long long range = 0;
  const unsigned long long* table = nullptr;
  const unsigned* bitmap = nullptr;  // presence bits (L2-resident filter)
  const long long* hkeys = nullptr;  // open addressing: keys per slot
  unsigned long long hmask = 0;
  const unsigned* mult = nullptr;    // weighted (1:N) builds: multiplicity per slot
  // row_rec builds (no table): the row is bits 32-63 of rowrec[slot * rstride]
  const unsigned long long* rowrec = nullptr;
  long long rstride = 0;
};

__device__ __forceinline__ unsigned long long build_hslot(long long key, unsigned long long mask) {
  unsigned long long h = static_cast<unsigned long long>(key) * 0x9E3779B97F4A7C15ULL;
  return (h ^ (h >> 31)) & mask;
}

// Branch-free predicate term for the fact scan: all compares on one column
// are merged into lo <= x <= hi (int64: one unsigned compare; fp64: two
// compares, NaN fails both exactly as the reference's `<`/`>` do).
enum RangeKind : int { RK_INT = 0, RK_F64 = 1, RK_INT_NE = 2, RK_F64_NE = 3, RK_TRUE = 4, RK_FALSE = 5 };
struct RTerm {
  int col = -1;
  int kind = RK_TRUE;
  unsigned long long lo = 0, hi = 0;  // bit patterns (int64 or fp64)
};

__device__ __forceinline__ bool eval_rterm(const RTerm& t, unsigned long long x) {
  switch (t.kind) {
    case RK_INT: return x - t.lo <= t.hi - t.lo;
    case RK_F64: {
      double d = __longlong_as_double(static_cast<long long>(x));
      return d >= __longlong_as_double(static_cast<long long>(t.lo)) &&
             d <= __longlong_as_double(static_cast<long long>(t.hi));
    }
    case RK_INT_NE: return x != t.lo;
    case RK_F64_NE:
      return __longlong_as_double(static_cast<long long>(x)) != __longlong_as_double(static_cast<long long>(t.lo));
    case RK_TRUE: return true;
    default: return false;
  }
}

// MODE_HASH group key: a fact column or a probe's root column. Every key
// maps to a digit (v - kmin) / step in [0, range) (int64 / date: step 86400e9
// for day-aligned dates; STR8 rows of width <= 7: the bytes big-endian, so
// digit order is the reference's byte order of zero-padded rows), and the
// group code is the mixed-radix number of the digits, first key most
// significant: ascending codes are the reference's ascending key order.
struct GKey {
  Operand x;
  int width = 0;  // 0: int64 / date; 1..7: STR8 bytes per row
  long long kmin = 0;
  long long step = 1;
  unsigned long long range = 1;
  unsigned long long stride = 1;
  // dictionary digit (wide int64 keys): rank of the value among the column's
  // distinct values, looked up in an open-addressing map (dkeys / dranks)
  const long long* dkeys = nullptr;
  const unsigned* dranks = nullptr;
  unsigned long long dmask = 0;
  long long dempty = 0;
};
constexpr unsigned long long kHashBusy = ~0ULL;       // tag of a slot being claimed
constexpr unsigned long long kCntAdd = 1ULL << 40;    // packed count: rows | adds << 40
constexpr unsigned long long kCntMask = kCntAdd - 1;

struct ProbeSpec {
  long long n = 0;
  int nterms = 0;
  RTerm terms[kMaxTerms];
  int nprobes = 0;
  Probe probes[kMaxProbes];
  int nacc = 0;
  Acc acc[kMaxAcc];
  int nkeys = 0;
  Operand keys[kMaxKeys];  // MODE_SMALL: 1-byte string columns (fact)
  int group_probe = -1;    // MODE_BUILDGRP
  // outputs
  unsigned long long* part;  // SCALAR: [cta][nacc+1]; SMALL: per-CTA tables
  // BUILDGRP group records, gstride words per group (a multiple of 4: whole
  // 32-byte sectors): [row count, kLimbWords limbs per accumulator]
  unsigned long long* gacc;  // record + 1
  unsigned long long* gcnt;  // record
  int gstride;
  unsigned* touched;         // BUILDGRP: bit per group with a row (the top-k walk's index)
  long long* err;            // [0] != 0: data violates the fused preconditions
  // MODE_HASH: group table of hcap slots; tag = code + 1 (0 empty,
  // kHashBusy while the claiming thread zeroes the slot's record); hdirect:
  // slot = code (the code range fits), else multiplicative hash + linear
  // probing; hpriv: the whole code range fits one CTA's shared memory (the
  // CTA accumulates there and flushes once)
  int nhkeys;
  GKey hkeys[kMaxKeys];
  unsigned long long* htag;
  unsigned long long hmask;
  int hdirect, hpriv;
  // weighted run (some build keys repeat): a row counts prod(mult) times;
  // probes whose root row is read (operands, keys, flags, groups) must match
  // exactly one build row (root_mask bit p), else the exact path
  int weighted;
  unsigned root_mask;
  // MODE_HASH: max |int64 value| over the scan (atomicMax); each group's
  // int sums are checked against it at output (max x rows < 2^63: no prefix
  // of the reference's sequential sum can overflow), not the whole scan's rows
  long long* absmax_out;
  int hflags;  // >= 0: record word of per-accumulator NaN / +Inf / -Inf bits (special run)
  int qfrac;          // MODE_HASH fixed-point fraction bits (64, or more after a re-run)
  long long* qstats;  // MODE_HASH: max of -(lowest set bit exponent) over unconvertible finite values
  // MODE_HASH sums as 2 limbs (l0 42-bit unsigned, l1 signed: v = l0 + l1 * 2^42)
  // while every value fits 105 bits; the reader checks per group that
  // adds < 2^22 and fmax x rows < 2^41 (else the unit re-runs with 3 limbs)
  int hlimbs;
  // word of accumulator a in a record (after the count word): 2-limb records
  // keep an int64 sum in ONE word (exact: the reader checks the scan's max
  // |value| x rows < 2^63 per group, so the wrapping add never wraps), an
  // fp64 sum in two limbs; 3-limb records: a * 3
  int hoff[kMaxAcc];
  long long* fmax_out;  // max |fp64 value| (bit pattern, atomicMax) over the scan
};

struct BuildSpec {
  long long n = 0;
  int nterms = 0;
  Term terms[kMaxTerms];
  int nstr = 0;
  StrTerm str[kMaxStrTerms];
  int nprobes = 0;
  Probe probes[kMaxProbes];
  int nflags = 0;
  StrTerm flags[kMaxFlags];
  Operand key;  // root key column (int64)
  long long kmin = 0;
  long long range = 0;
  unsigned long long* table = nullptr;
  unsigned* bitmap = nullptr;
  long long* hkeys = nullptr;  // open-addressing build (see Probe)
  unsigned long long hmask = 0;
  unsigned* mult = nullptr;    // weighted build: summed row weights per slot
  int assign_groups = 0;
  // group records zeroed by the row inserted into the slot (no memset over
  // the whole key range): zrec_words words per slot (whole sectors)
  unsigned long long* zrec = nullptr;
  int zrec_words = 0;
  long long* err = nullptr;
  // the key column holds no repeated value (KeyRange::unique): presence bits
  // are set fire-and-forget, nothing to check (presence_insert_unique)
  int unique = 0;
  // a flagless group-assigning build keeps the row in its record's count
  // word (bits 32-63 = row + 1) instead of a table entry: one 32-byte
  // sector written per inserted row instead of two
  int row_rec = 0;
};

// Presence bits of one insert round of a warp. Sparse rounds (few lanes
// inserting, e.g. Q3's orders build at a 10 % pass rate) issue one atomicOr
// per row; dense rounds (every row of an unfiltered build, e.g. Q14's part)
// first OR-reduce the lanes that share a word (__match_any_sync) so one
// lane sets them - per-row atomics there would hit one word 32 times. Two
// inserted rows with one key (a 1:N join, outside the fused contract) show
// up as a bit the word already held, or inside a dense round as fewer bits
// than lanes; the atomic's old word is returned in `old` (with the bits in
// `set`) and only checked by build_dup_check after the thread's last round,
// so no round waits on the atomic's return. Orders build 110 -> 104 us with
// the sparse form; the part build keeps the dense one.
__device__ __forceinline__ void presence_insert(unsigned* bitmap, long long idx, unsigned& old, unsigned& set,
                                                unsigned& dup) {
  old = 0u;
  set = 0u;
  const unsigned active = __ballot_sync(0xffffffffu, idx >= 0);
  if (__popc(active) < 8) {  // warp-uniform
    if (idx >= 0) {
      set = 1u << (idx & 31);
      old = atomicOr(bitmap + (idx >> 5), set);
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const unsigned word = idx >= 0 ? static_cast<unsigned>(idx >> 5) : 0xffffffffu;
  const unsigned peers = __match_any_sync(0xffffffffu, word);
  const unsigned bits = __reduce_or_sync(peers, idx >= 0 ? 1u << (idx & 31) : 0u);
  if (idx >= 0 && lane == __ffs(peers) - 1) {
    old = atomicOr(bitmap + word, bits);
    set = bits;
    dup |= __popc(bits) != __popc(peers) ? 1u : 0u;
  }
}
// Presence bits over a key column known to hold no repeated value: the same
// sparse / warp-aggregated rounds as presence_insert, but the old words are
// never needed, so the atomics do not return (RED) and no thread waits on one
// (Q3's orders build: the wait on the returned words at the end of every
// thread was part of its latency chain).
__device__ __forceinline__ void presence_insert_unique(unsigned* bitmap, long long idx) {
  const unsigned active = __ballot_sync(0xffffffffu, idx >= 0);
  if (__popc(active) < 8) {  // warp-uniform
    if (idx >= 0) atomicOr(bitmap + (idx >> 5), 1u << (idx & 31));
    return;
  }
  const int lane = threadIdx.x & 31;
  const unsigned word = idx >= 0 ? static_cast<unsigned>(idx >> 5) : 0xffffffffu;
  const unsigned peers = __match_any_sync(0xffffffffu, word);
  const unsigned bits = __reduce_or_sync(peers, idx >= 0 ? 1u << (idx & 31) : 0u);
  if (idx >= 0 && lane == __ffs(peers) - 1) atomicOr(bitmap + word, bits);
}
__device__ __forceinline__ void set_fallback(long long* err, long long reason) {
  atomicExch(reinterpret_cast<unsigned long long*>(err), 1ULL);
  atomicExch(reinterpret_cast<unsigned long long*>(err) + 3, static_cast<unsigned long long>(reason));
}
__device__ __forceinline__ void build_dup_check(unsigned dup, long long* err) {
  if (__any_sync(0xffffffffu, dup != 0u) && (threadIdx.x & 31) == 0) set_fallback(err, FR_DUP_KEY);
}

// ---- operand access ----------------------------------------------------------
__device__ __forceinline__ long long ld_i64(const void* p, long long r) {
  return __ldg(static_cast<const long long*>(p) + r);
}
__device__ __forceinline__ double ld_f64(const void* p, long long r) {
  return __ldg(static_cast<const double*>(p) + r);
}

// two consecutive fact rows (row0 even) with one 128-bit load
__device__ __forceinline__ void ld_pair(const Operand& o, long long row0, unsigned long long& a,
                                        unsigned long long& b) {
  if (o.type == OT_U8) {
    unsigned short v = __ldg(reinterpret_cast<const unsigned short*>(static_cast<const uint8_t*>(o.ptr) + row0));
    a = v & 0xff;
    b = v >> 8;
  } else {
    ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(static_cast<const unsigned long long*>(o.ptr) + row0));
    a = v.x;
    b = v.y;
  }
}

__device__ __forceinline__ unsigned long long ld_row(const Operand& o, long long row) {
  if (o.type == OT_U8) return __ldg(static_cast<const uint8_t*>(o.ptr) + row);
  return __ldg(static_cast<const unsigned long long*>(o.ptr) + row);
}

template <typename T>
__device__ __forceinline__ bool cmp_op(T x, T y, int op) {
  switch (op) {
    case TQP_EQ: return x == y;
    case TQP_NE: return x != y;
    case TQP_LT: return x < y;
    case TQP_LE: return x <= y;
    case TQP_GT: return x > y;
    default: return x >= y;
  }
}

__device__ __forceinline__ bool eval_term(const Term& t, unsigned long long raw) {
  switch (t.kind) {
    case TK_INT: return cmp_op<long long>(static_cast<long long>(raw), t.ik, t.op);
    case TK_F64: return cmp_op<double>(__longlong_as_double(static_cast<long long>(raw)), t.fk, t.op);
    case TK_TRUE: return true;
    default: return false;
  }
}

__device__ __forceinline__ bool eval_str(const StrTerm& s, long long row) {
  const uint8_t* p = s.ptr + row * s.width;
  int len = 0;
  while (len < s.width && p[len] != 0) ++len;
  if (s.is_like) {
    int pl = s.litlen;
    if (pl > len) return false;
    auto at = [&](int off) {
      for (int j = 0; j < pl; ++j)
        if (p[off + j] != s.lit[j]) return false;
      return true;
    };
    switch (s.anchor) {
      case TQP_START: return at(0);
      case TQP_END: return at(len - pl);
      case TQP_ANY:
        for (int o = 0; o + pl <= len; ++o)
          if (at(o)) return true;
        return false;
      default: return len == pl && at(0);
    }
  }
  int m = s.width > s.litlen ? s.width : s.litlen;
  int c = 0;
  for (int j = 0; j < m && c == 0; ++j) {
    int x = j < s.width ? p[j] : 0;
    int y = j < s.litlen ? s.lit[j] : 0;
    if (x != y) c = x < y ? -1 : 1;
  }
  return cmp_op<int>(c, 0, s.op);
}

__device__ __forceinline__ double apply_factor(const Factor& f, double x) {
  switch (f.kind) {
    case FK_X: return x;
    case FK_K_MINUS_X: return __dsub_rn(f.k, x);
    case FK_K_PLUS_X: return __dadd_rn(f.k, x);
    case FK_X_MINUS_K: return __dsub_rn(x, f.k);
    case FK_X_PLUS_K: return __dadd_rn(x, f.k);
    case FK_X_TIMES_K: return __dmul_rn(x, f.k);
    default: return f.k;
  }
}

struct RowCtx {
  long long rid[kMaxProbes];
  unsigned flags[kMaxProbes];
  unsigned gid[kMaxProbes];
  unsigned mult[kMaxProbes];
};

__device__ __forceinline__ bool probe_lookup(const Probe& p, long long key, long long& rid, unsigned& flags,
                                             unsigned& gid, unsigned* mult = nullptr) {
  long long idx;
  if (p.hkeys) {
    unsigned long long sl = build_hslot(key, p.hmask);
    const long long empty = p.kmin - 1;
    for (;;) {
      const long long k = __ldg(p.hkeys + sl);
      if (k == key) break;
      if (k == empty) return false;
      sl = (sl + 1) & p.hmask;
    }
    idx = static_cast<long long>(sl);
  } else {
    idx = key - p.kmin;
    if (idx < 0 || idx >= p.range) return false;
    if (p.bitmap && !((__ldg(p.bitmap + (idx >> 5)) >> (idx & 31)) & 1u)) return false;
  }
  unsigned long long e = p.table ? __ldg(p.table + idx) : p.rowrec[idx * p.rstride] >> 32;
  if (!e) return false;
  rid = static_cast<long long>(e & 0xffffffffULL) - 1;
  gid = static_cast<unsigned>(idx);  // a group-assigning build's group is its key slot
  flags = static_cast<unsigned>(e >> 57);
  if (mult) *mult = p.mult ? __ldg(p.mult + idx) : 1u;
  return true;
}

// open-addressing insert of `key` (build side): the slot, and whether the key
// was already there (a repeated build key)
__device__ __forceinline__ long long build_hash_insert(const BuildSpec& s, long long key, bool& seen) {
  unsigned long long sl = build_hslot(key, s.hmask);
  const unsigned long long empty = static_cast<unsigned long long>(s.kmin - 1);
  for (unsigned long long i = 0; i <= s.hmask; ++i) {
    const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(s.hkeys) + sl, empty,
                                             static_cast<unsigned long long>(key));
    if (old == empty || old == static_cast<unsigned long long>(key)) {
      seen = old != empty;
      return static_cast<long long>(sl);
    }
    sl = (sl + 1) & s.hmask;
  }
  return -1;
}

__device__ __forceinline__ unsigned long long operand_value(const Operand& o, unsigned long long fact_raw,
                                                            const RowCtx& rc) {
  if (o.src < 0) return fact_raw;
  return ld_row(o, rc.rid[o.src]);
}

// value of accumulator a for one row; fact operands already loaded in fv[]
__device__ __forceinline__ unsigned long long eval_acc(const Acc& a, const unsigned long long* fv, const RowCtx& rc) {
  if (a.is_int) return operand_value(a.f[0].x, fv[0], rc);
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < kMaxFactors; ++i) {
    if (i < a.nf) {
      double x = __longlong_as_double(static_cast<long long>(operand_value(a.f[i].x, fv[i], rc)));
      double y = apply_factor(a.f[i], x);
      v = i == 0 ? y : __dmul_rn(v, y);
    }
  }
  if (a.gate_probe >= 0 && !((rc.flags[a.gate_probe] >> a.gate_bit) & 1u)) v = a.gate_else;
  return static_cast<unsigned long long>(__double_as_longlong(v));
}

// ---- exact Q64.64 fixed point ----------------------------------------------------
// x -> x * 2^64 as int128, exactly: false for NaN, Inf, |x| >= 2^62 and for
// any x with a nonzero bit below 2^-64 (it would be truncated), so a group
// sum built from these values is exact or the unit falls back (FR_Q64_*).
// Every money value (a multiple of 2^-40 or coarser) converts.
// Q(128-F).F generalisation (F fraction bits; MODE_HASH re-runs with F > 64
// when a value has bits below 2^-64): exact or false
__device__ __forceinline__ bool f64_to_qf(double x, int F, __int128& out) {
  long long bits = __double_as_longlong(x);
  int ex = static_cast<int>((bits >> 52) & 0x7ff);
  if (ex == 0x7ff) return false;
  unsigned long long mant = static_cast<unsigned long long>(bits) & ((1ULL << 52) - 1);
  if (ex == 0) {
    ex = 1;
  } else {
    mant |= 1ULL << 52;
  }
  int shift = ex - 1075 + F;
  unsigned __int128 v;
  if (shift >= 0) {
    if (shift > 73) return false;
    v = static_cast<unsigned __int128>(mant) << shift;
  } else if (shift > -64) {
    if (mant & ((1ULL << (-shift)) - 1)) return false;  // bits below 2^-64
    v = static_cast<unsigned __int128>(mant >> (-shift));
  } else {
    if (mant) return false;
    v = 0;
  }
  out = bits < 0 ? -static_cast<__int128>(v) : static_cast<__int128>(v);
  return true;
}
__device__ __forceinline__ bool f64_to_q64(double x, __int128& out) { return f64_to_qf(x, 64, out); }

// binary exponent of the lowest set bit of a finite nonzero x
__device__ __forceinline__ int lowbit_exp(double x) {
  const long long bits = __double_as_longlong(x);
  int ex = static_cast<int>((bits >> 52) & 0x7ff);
  unsigned long long mant = static_cast<unsigned long long>(bits) & ((1ULL << 52) - 1);
  if (ex == 0) ex = 1;
  else mant |= 1ULL << 52;
  return ex - 1075 + (mant ? __ffsll(static_cast<long long>(mant)) - 1 : 0);
}

// Q64.64 group sums cannot wrap while max|value| x rows < 2^62 (the limb
// words are bounded separately by kLimbMaxRows); checked once per thread
// after its last row with the largest |value| it converted
__device__ __forceinline__ void q64_range_check(double fabsmax, long long rows, long long* err, int F = 64) {
  if (fabsmax * static_cast<double>(rows) >= ldexp(4.6116860184273879e18, 64 - F)) set_fallback(err, FR_Q64_RANGE);
}

// Q64.64 -> fp64, correctly rounded (one rounding of the exact value: the
// int128 conversion rounds to nearest even, the 2^-64 scale is exact)
// int128 -> fp64 rounded to nearest even: the top 64 significant bits with
// every lower bit folded into their last (sticky) bit round exactly like
// the whole value (11 spare bits below the double's 53), one 64-bit convert
__device__ __forceinline__ double i128_to_f64_rn(__int128 v) {
  const long long lo64 = static_cast<long long>(v);
  if (static_cast<__int128>(lo64) == v) return static_cast<double>(lo64);
  const bool neg = v < 0;
  const unsigned __int128 u = neg ? static_cast<unsigned __int128>(0) - static_cast<unsigned __int128>(v)
                                  : static_cast<unsigned __int128>(v);
  const unsigned long long uh = static_cast<unsigned long long>(u >> 64), ul = static_cast<unsigned long long>(u);
  unsigned long long top;
  int e;  // u = top * 2^e (+ sticky bits)
  if (uh == 0) {
    top = ul;
    e = 0;
  } else {
    const int lz = __clzll(static_cast<long long>(uh));
    top = lz ? (uh << lz) | (ul >> (64 - lz)) : uh;
    const unsigned long long rest = lz ? (ul << lz) : ul;
    top |= rest != 0 ? 1ULL : 0ULL;
    e = 64 - lz;
  }
  const double d = ldexp(__ull2double_rn(top), e);
  return neg ? -d : d;
}

__device__ __forceinline__ double q64_to_f64(unsigned long long lo, unsigned long long hi) {
  const __int128 v = static_cast<__int128>((static_cast<unsigned __int128>(hi) << 64) | lo);
  return i128_to_f64_rn(v) * 5.421010862427522e-20;  // 2^-64
}

__device__ __forceinline__ void atomic_add_q64(unsigned long long* p, __int128 v) {
  unsigned long long lo = static_cast<unsigned long long>(v);
  unsigned long long hi = static_cast<unsigned long long>(static_cast<unsigned __int128>(v) >> 64);
  unsigned long long old = atomicAdd(p, lo);
  unsigned long long carry = (old + lo < old) ? 1ULL : 0ULL;
  atomicAdd(p + 1, hi + carry);
}

// Carry-free group sums: an int128 is added as three 42-bit limbs
// (v = l0 + l1 * 2^42 + l2 * 2^84, l0/l1 unsigned, l2 signed) with three
// non-returning atomic adds, so no thread waits on an atomic's return value.
// A word takes < 2^21 adds of < 2^42 without overflow; the reader checks the
// group's row count against kLimbMaxRows and reassembles mod 2^128 (exact
// whenever the true sum fits, as the int128 it replaces).
constexpr int kLimbWords = 3;
constexpr long long kLimbMaxRows = 1LL << 21;
__device__ __forceinline__ void atomic_add_limbs(unsigned long long* p, __int128 v) {
  const unsigned __int128 u = static_cast<unsigned __int128>(v);
  const unsigned long long m = (1ULL << 42) - 1;
  atomicAdd(p, static_cast<unsigned long long>(u) & m);
  atomicAdd(p + 1, static_cast<unsigned long long>(u >> 42) & m);
  atomicAdd(p + 2, static_cast<unsigned long long>(static_cast<long long>(v >> 84)));
}
// 2-limb form (MODE_HASH): false if v needs more than 105 bits
__device__ __forceinline__ bool atomic_add_limbs2(unsigned long long* p, __int128 v, unsigned long long pol) {
  const __int128 hi = v >> 42;
  if (hi != static_cast<__int128>(static_cast<long long>(hi))) return false;
  unsigned long long lo = static_cast<unsigned long long>(v) & ((1ULL << 42) - 1);
  unsigned long long h = static_cast<unsigned long long>(static_cast<long long>(hi));
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(lo), "l"(pol) : "memory");
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p + 1), "l"(h), "l"(pol) : "memory");
  return true;
}
__device__ __forceinline__ __int128 limbs2_to_i128(const unsigned long long* w) {
  return static_cast<__int128>(static_cast<unsigned __int128>(w[0]) +
                               static_cast<unsigned __int128>(static_cast<__int128>(static_cast<long long>(w[1])) << 42));
}
__device__ __forceinline__ __int128 limbs_to_i128(const unsigned long long* w) {
  const unsigned __int128 u = static_cast<unsigned __int128>(w[0]) + (static_cast<unsigned __int128>(w[1]) << 42) +
                              (static_cast<unsigned __int128>(static_cast<__int128>(static_cast<long long>(w[2]))) << 84);
  return static_cast<__int128>(u);
}

// ---- MODE_HASH group table --------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// digit of key K for one row: `raw` is the loaded int64 (width 0); STR8 keys
// read their `width` bytes at `row` (big-endian, so digit order = byte order)
__device__ __forceinline__ unsigned long long gkey_digit(const GKey& K, unsigned long long raw, long long row) {
  if (K.width) {
    const uint8_t* p = static_cast<const uint8_t*>(K.x.ptr) + row * K.width;
    unsigned long long d = 0;
    for (int j = 0; j < K.width; ++j) d = (d << 8) | __ldg(p + j);
    if (!K.dkeys) return d;
    raw = d;  // dictionary over the packed rows
  }
  if (K.dkeys) {
    const long long v = static_cast<long long>(raw);
    unsigned long long h = static_cast<unsigned long long>(v) * 0x9E3779B97F4A7C15ULL;
    unsigned long long sl = (h ^ (h >> 31)) & K.dmask;
    for (;;) {
      const long long k = __ldg(K.dkeys + sl);
      if (k == v) return __ldg(K.dranks + sl);
      if (k == K.dempty) return ~0ULL;  // not in the dictionary: flagged as out of range
      sl = (sl + 1) & K.dmask;
    }
  }
  unsigned long long d = raw - static_cast<unsigned long long>(K.kmin);
  if (K.step != 1) d /= static_cast<unsigned long long>(K.step);
  return d;
}

// slot of group `code` in the global table, claimed (record zeroed, then the
// tag published) by the first row that meets it; -1: table full
__device__ __forceinline__ long long hash_claim(const ProbeSpec& s, unsigned long long code) {
  const unsigned long long want = code + 1;
  unsigned long long slot = code;
  if (!s.hdirect) {
    unsigned long long h = code * 0x9E3779B97F4A7C15ULL;
    slot = (h ^ (h >> 29)) & s.hmask;
  }
  for (unsigned long long probe = 0; probe <= s.hmask; ++probe) {
    unsigned long long* tp = s.htag + slot;
    unsigned long long t = ld_acquire_u64(tp);
    if (t == 0ULL) {
      t = atomicCAS(tp, 0ULL, kHashBusy);
      if (t == 0ULL) {
        unsigned long long* rec = s.gcnt + static_cast<long long>(slot) * s.gstride;
        for (int w = 0; w < s.gstride; ++w) rec[w] = 0ULL;
        __threadfence();
        atomicExch(tp, want);
        return static_cast<long long>(slot);
      }
    }
    while (t == kHashBusy) t = ld_acquire_u64(tp);
    if (t == want) return static_cast<long long>(slot);
    slot = (slot + 1) & s.hmask;
  }
  return -1;
}

// ---- TMA-staged, warp-specialised tile pipeline for the fact scan -----------
// A persistent CTA per SM streams tiles of kTileRows rows. Warp 0 is the
// producer: one lane issues, for every distinct fact column, a 1-D bulk async
// copy (cp.async.bulk.shared::cluster.global -> SASS UBLKCP) of the tile into
// a multi-stage shared-memory ring, signalling a `full` mbarrier with the
// expected transaction bytes. Warps 1..16 consume: wait on `full`, evaluate
// their rows, arrive on the stage's `empty` mbarrier. There is no CTA-wide
// barrier per tile, ~100-190 KB per SM stay in flight independent of register
// use, and operands are addressed by runtime column index in shared memory.
// Predicates, probes and accumulator expressions run as compact runtime
// loops whose dispatch is amortised over the rows each thread owns.
constexpr int kTileRows = 2048;  // 16 KB bulk copies per 8-byte column
constexpr int kMaxStages = 8;
constexpr int kMaxCols = 10;

// consumer warps per mode (+1 producer warp): small-group keeps 48 register
// accumulators per thread, so it runs fewer, wider threads
template <int MODE, bool LEAN = false>
struct TileShape {
  // small-group keeps per-thread shared-memory accumulators (groups x
  // accumulators x threads), so its tiles are half as tall. The lean
  // hash-group instance (LEAN) has the same shape: 24 or 28 consumer warps
  // (2 rows per thread) ran its scan 3-7 % slower than 16 (qg at SF10)
  static constexpr int ROWS = MODE == MODE_SMALL ? 1024 : kTileRows;  // MODE_HASH: as SCALAR
  static constexpr int CW = MODE == MODE_SMALL ? 8 : 16;
  static constexpr int CT = CW * 32;
  static constexpr int THREADS = CT + 32;
  static constexpr int R = ROWS / CT;  // rows per consumer thread
  static constexpr int SUB = R;
  static_assert(ROWS % CT == 0, "a tile is a whole number of rows per consumer thread");
};

struct TileSpec {
  ProbeSpec p;
  int ncols = 0;
  const unsigned char* col_ptr[kMaxCols];
  int col_w[kMaxCols];
  int col_off[kMaxCols];  // byte offset of the column inside a stage
  int stage_bytes = 0;
  int stages = 3;
  int rows = kTileRows;   // rows per tile
  int aux_bytes = 0;      // per-thread accumulator / staging region
  int evict_first = 0;    // stream the fact tiles with an L2 evict-first policy (keeps a
                          // hash-group table resident in L2 under the stream)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// non-returning u64 add with an L2 cache policy (hash-group table words)
__device__ __forceinline__ void red_add_hint(unsigned long long* p, unsigned long long v, unsigned long long pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// HINT: the copies carry an L2 evict-first policy (hash-group scans, which
// keep their table resident under the stream); a compile-time choice, so the
// other pipelines' producer loop is exactly the unhinted one
template <bool HINT = false>
__device__ __forceinline__ void issue_tile(const TileSpec& t, unsigned char* stage, unsigned long long* bar,
                                           long long tile) {
  const long long row0 = tile * t.rows;
  long long rows = t.p.n - row0;
  if (rows > t.rows) rows = t.rows;
  unsigned total = 0;
  for (int c = 0; c < t.ncols; ++c) total += static_cast<unsigned>((rows * t.col_w[c] + 15) & ~15LL);
  mbar_expect_tx(bar, total);
  for (int c = 0; c < t.ncols; ++c) {
    unsigned bytes = static_cast<unsigned>((rows * t.col_w[c] + 15) & ~15LL);
    if constexpr (HINT) bulk_g2s_hint(stage + t.col_off[c], t.col_ptr[c] + row0 * t.col_w[c], bytes, bar, l2_policy_evict_first());
    else bulk_g2s(stage + t.col_off[c], t.col_ptr[c] + row0 * t.col_w[c], bytes, bar);
  }
}

__device__ __forceinline__ unsigned long long add_acc(bool is_int, unsigned long long a, unsigned long long b) {
  if (is_int) return static_cast<unsigned long long>(static_cast<long long>(a) + static_cast<long long>(b));
  return static_cast<unsigned long long>(__double_as_longlong(
      __dadd_rn(__longlong_as_double(static_cast<long long>(a)), __longlong_as_double(static_cast<long long>(b)))));
}

struct SmallPart {  // MODE_SMALL per-CTA partial, in global memory
  unsigned int codes[kGroups];
  unsigned long long cnt[kGroups];
  unsigned long long acc[kGroups][kMaxAcc];
};

__device__ __forceinline__ unsigned hash_code(unsigned c) { return (c * 2654435761u) >> (32 - kGroupBits); }

// per-thread region: SCALAR running sums [acc][thread]; SMALL accumulators
// [group][acc + count][thread]
template <int MODE>
__host__ __device__ constexpr size_t aux_bytes_for(int nacc) {
  using S = TileShape<MODE>;
  return MODE == MODE_SMALL ? sizeof(unsigned long long) * kGroups * (nacc + 1) * S::CT : 0;
}

}  // namespace fz
}  // namespace tqp
