/* tqp_gen.h — counter-based TPC-H-shaped data generator (host C/C++ and CUDA).
 *
 * The reference ships no generator (its CLI is `int main(){return 0;}`,
 * /root/reference/proj/tools/placeholder.cpp:1); its distributions exist only
 * as prose at /root/reference/SPEC.md:601 (lineitem/part). This header
 * restates those distributions and extends them for Q1/Q3:
 * every value is a pure function of (seed, stream, index) through SplitMix64,
 * so any shard can be generated independently and the CPU oracle and every
 * GPU count see bit-identical bytes.
 *
 *   orders   o_orderkey 1..N_o, o_custkey U{1..150000*SF},
 *            o_orderdate U[1992-01-01, 1998-08-02], o_shippriority 0,
 *            lines per order U{1..7}; lineitem rows = round(6e6*SF) exactly
 *            (the last order is truncated), emitted in orderkey order.
 *   lineitem l_orderkey, l_partkey U{1..200000*SF}, l_quantity U{1..50},
 *            l_extendedprice = U{90000..10500000} cents / 100.0,
 *            l_discount = U{0..10}/100.0, l_tax = U{0..8}/100.0,
 *            l_shipdate = o_orderdate + U{1..121} days,
 *            receipt = l_shipdate + U{1..30} days (not stored),
 *            l_returnflag = receipt <= 1995-06-17 ? ('R'|'A' 50/50) : 'N',
 *            l_linestatus = l_shipdate > 1995-06-17 ? 'O' : 'F'.
 *   part     p_partkey 1..200000*SF, p_type = "<p1> <p2> <p3>" (6x5x5 words).
 *   customer c_custkey 1..150000*SF, c_mktsegment uniform over 5 segments.
 *
 * Money is emitted as cents/100.0 and rates as k/100.0: both are correctly
 * rounded, hence bit-identical to what the reference's CSV parser
 * (std::from_chars, columnar.cpp:403-409) and SQL literal parser (std::stod,
 * sql_parser.cpp:245-247) produce for the same decimal text.
 */
#ifndef TQP_GEN_H
#define TQP_GEN_H

#include <stdint.h>

#ifdef __CUDACC__
#define TQP_HD __host__ __device__ __forceinline__
#else
#define TQP_HD static inline
#endif

#define TQP_NS_PER_DAY 86400000000000LL

enum tqp_gen_stream {
  TQP_S_ORD_LINES = 1,
  TQP_S_ORD_CUST = 2,
  TQP_S_ORD_DATE = 3,
  TQP_S_L_PART = 10,
  TQP_S_L_QTY = 11,
  TQP_S_L_PRICE = 12,
  TQP_S_L_DISC = 13,
  TQP_S_L_TAX = 14,
  TQP_S_L_SHIP = 15,
  TQP_S_L_RECEIPT = 16,
  TQP_S_L_RFLAG = 17,
  TQP_S_P_TYPE = 20,
  TQP_S_C_SEG = 30
};

TQP_HD uint64_t tqp_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* Uniform 64-bit draw for element `i` of stream `stream`. */
TQP_HD uint64_t tqp_draw(uint64_t seed, uint32_t stream, uint64_t i) {
  uint64_t key = tqp_splitmix64(seed ^ (0xA0761D6478BD642FULL * (uint64_t)stream));
  return tqp_splitmix64(key + i * 0xE7037ED1A0B428DBULL);
}

/* Uniform integer in [lo, hi] (inclusive). */
TQP_HD int64_t tqp_uniform(uint64_t seed, uint32_t stream, uint64_t i, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1ULL;
  return lo + (int64_t)(tqp_draw(seed, stream, i) % span);
}

/* Days since 1970-01-01 of a proleptic-Gregorian civil date (same arithmetic
 * contract as tensql::days_from_civil, columnar.hpp:60). */
TQP_HD int64_t tqp_days_from_civil(int64_t y, int64_t m, int64_t d) {
  y -= m <= 2;
  int64_t era = (y >= 0 ? y : y - 399) / 400;
  int64_t yoe = y - era * 400;
  int64_t doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
  int64_t doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + doe - 719468;
}

/* Scale-factor cardinalities. */
TQP_HD int64_t tqp_round_sf(double base, double sf) {
  double v = base * sf;
  return (int64_t)(v + 0.5);
}
TQP_HD int64_t tqp_lineitem_rows(double sf) { return tqp_round_sf(6000000.0, sf); }
TQP_HD int64_t tqp_part_rows(double sf) { return tqp_round_sf(200000.0, sf); }
TQP_HD int64_t tqp_customer_rows(double sf) { return tqp_round_sf(150000.0, sf); }

/* ---- orders -------------------------------------------------------------- */
TQP_HD int32_t tqp_order_lines(uint64_t seed, int64_t orderkey) {
  return (int32_t)tqp_uniform(seed, TQP_S_ORD_LINES, (uint64_t)orderkey, 1, 7);
}
TQP_HD int64_t tqp_o_custkey(uint64_t seed, double sf, int64_t orderkey) {
  int64_t nc = tqp_customer_rows(sf);
  return tqp_uniform(seed, TQP_S_ORD_CUST, (uint64_t)orderkey, 1, nc > 0 ? nc : 1);
}
/* o_orderdate in days since epoch: U[1992-01-01, 1998-08-02]. */
TQP_HD int64_t tqp_o_orderdate_days(uint64_t seed, int64_t orderkey) {
  int64_t lo = tqp_days_from_civil(1992, 1, 1);
  int64_t hi = tqp_days_from_civil(1998, 8, 2);
  return tqp_uniform(seed, TQP_S_ORD_DATE, (uint64_t)orderkey, lo, hi);
}

/* ---- lineitem (row index r is the global row number; orderkey/date come
 * from the owning order) --------------------------------------------------- */
TQP_HD int64_t tqp_l_partkey(uint64_t seed, double sf, int64_t r) {
  int64_t np = tqp_part_rows(sf);
  return tqp_uniform(seed, TQP_S_L_PART, (uint64_t)r, 1, np > 0 ? np : 1);
}
TQP_HD int64_t tqp_l_quantity(uint64_t seed, int64_t r) {
  return tqp_uniform(seed, TQP_S_L_QTY, (uint64_t)r, 1, 50);
}
TQP_HD double tqp_l_extendedprice(uint64_t seed, int64_t r) {
  return (double)tqp_uniform(seed, TQP_S_L_PRICE, (uint64_t)r, 90000, 10500000) / 100.0;
}
TQP_HD double tqp_l_discount(uint64_t seed, int64_t r) {
  return (double)tqp_uniform(seed, TQP_S_L_DISC, (uint64_t)r, 0, 10) / 100.0;
}
TQP_HD double tqp_l_tax(uint64_t seed, int64_t r) {
  return (double)tqp_uniform(seed, TQP_S_L_TAX, (uint64_t)r, 0, 8) / 100.0;
}
TQP_HD int64_t tqp_l_shipdate_days(uint64_t seed, int64_t r, int64_t orderdate_days) {
  return orderdate_days + tqp_uniform(seed, TQP_S_L_SHIP, (uint64_t)r, 1, 121);
}
/* Returns the flag byte ('R', 'A' or 'N'). */
TQP_HD uint8_t tqp_l_returnflag(uint64_t seed, int64_t r, int64_t shipdate_days) {
  int64_t receipt = shipdate_days + tqp_uniform(seed, TQP_S_L_RECEIPT, (uint64_t)r, 1, 30);
  if (receipt <= tqp_days_from_civil(1995, 6, 17)) {
    return (tqp_draw(seed, TQP_S_L_RFLAG, (uint64_t)r) & 1ULL) ? (uint8_t)'R' : (uint8_t)'A';
  }
  return (uint8_t)'N';
}
TQP_HD uint8_t tqp_l_linestatus(int64_t shipdate_days) {
  return shipdate_days > tqp_days_from_civil(1995, 6, 17) ? (uint8_t)'O' : (uint8_t)'F';
}

/* ---- part / customer strings --------------------------------------------- */
#define TQP_P_TYPE_WIDTH 25
#define TQP_C_SEG_WIDTH 10

/* Writes p_type of part row p (0-based; p_partkey = p+1) into out[0..25),
 * zero padded; returns the byte length. Prefix PROMO has share 1/6. */
TQP_HD int tqp_p_type(uint64_t seed, int64_t p, uint8_t* out) {
  const char* w1[6] = {"PROMO", "STANDARD", "SMALL", "MEDIUM", "ECONOMY", "LARGE"};
  const char* w2[5] = {"ANODIZED", "BURNISHED", "PLATED", "POLISHED", "BRUSHED"};
  const char* w3[5] = {"TIN", "NICKEL", "BRASS", "STEEL", "COPPER"};
  uint64_t d = tqp_draw(seed, TQP_S_P_TYPE, (uint64_t)p);
  const char* parts[3] = {w1[d % 6], w2[(d / 6) % 5], w3[(d / 30) % 5]};
  int n = 0;
  for (int k = 0; k < 3; ++k) {
    if (k) out[n++] = (uint8_t)' ';
    for (const char* c = parts[k]; *c; ++c) out[n++] = (uint8_t)*c;
  }
  for (int j = n; j < TQP_P_TYPE_WIDTH; ++j) out[j] = 0;
  return n;
}

/* Writes c_mktsegment of customer row c (0-based) into out[0..10). */
TQP_HD int tqp_c_mktsegment(uint64_t seed, int64_t c, uint8_t* out) {
  const char* segs[5] = {"AUTOMOBILE", "BUILDING", "FURNITURE", "HOUSEHOLD", "MACHINERY"};
  const char* s = segs[tqp_draw(seed, TQP_S_C_SEG, (uint64_t)c) % 5];
  int n = 0;
  for (; s[n]; ++n) out[n] = (uint8_t)s[n];
  for (int j = n; j < TQP_C_SEG_WIDTH; ++j) out[j] = 0;
  return n;
}

#endif /* TQP_GEN_H */
