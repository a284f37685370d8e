// Device-side TPC-H generator: the same counter-based functions as
// include/tqp_gen.h (host and device share the header), so device tables are
// bit-identical to the tables the CPU oracle builds
// (oracle/tools/tpch_tables.hpp). lineitem/orders shards are cut on order
// boundaries (every order's lines land on one shard).
#include <cmath>
#include <string>

#include "executor.hpp"
#include "device.cuh"
#include "tqp_gen.h"

namespace tqp {
namespace {

__global__ void k_order_lines(uint64_t seed, int64_t n, int64_t* __restrict__ out) {
  for (int64_t o = gtid(); o < n; o += gstride()) out[o] = tqp_order_lines(seed, o + 1);
}

// first index i in [0,n) with offs[i] >= target (offs non-decreasing)
__global__ void k_lower_bounds(const int64_t* __restrict__ offs, int64_t n, const int64_t* __restrict__ targets,
                               int64_t nt, int64_t* __restrict__ out) {
  for (int64_t t = gtid(); t < nt; t += gstride()) {
    int64_t a = 0, b = n;
    while (a < b) {
      int64_t m = (a + b) >> 1;
      if (offs[m] < targets[t]) a = m + 1;
      else b = m;
    }
    out[t] = a;
  }
}

struct LineitemCols {
  int64_t *okey, *pkey, *qty, *ship;
  double *price, *disc, *tax;
  uint8_t *rflag, *lstatus;
};

__global__ void k_gen_lineitem(uint64_t seed, double sf, const int64_t* __restrict__ offs, int64_t o_lo, int64_t o_hi,
                               int64_t L, int64_t row_lo, LineitemCols c) {
  for (int64_t o = o_lo + gtid(); o < o_hi; o += gstride()) {
    int64_t ok = o + 1;
    int64_t od = tqp_o_orderdate_days(seed, ok);
    int64_t a = offs[o], b = a + tqp_order_lines(seed, ok);
    if (b > L) b = L;
    for (int64_t r = a; r < b; ++r) {
      int64_t i = r - row_lo;
      int64_t sd = tqp_l_shipdate_days(seed, r, od);
      c.okey[i] = ok;
      c.pkey[i] = tqp_l_partkey(seed, sf, r);
      c.qty[i] = tqp_l_quantity(seed, r);
      c.price[i] = tqp_l_extendedprice(seed, r);
      c.disc[i] = tqp_l_discount(seed, r);
      c.tax[i] = tqp_l_tax(seed, r);
      c.ship[i] = sd * TQP_NS_PER_DAY;
      c.rflag[i] = tqp_l_returnflag(seed, r, sd);
      c.lstatus[i] = tqp_l_linestatus(sd);
    }
  }
}

__global__ void k_gen_orders(uint64_t seed, double sf, int64_t o_lo, int64_t o_hi, int64_t* __restrict__ okey,
                             int64_t* __restrict__ cust, int64_t* __restrict__ date, int64_t* __restrict__ prio) {
  for (int64_t o = o_lo + gtid(); o < o_hi; o += gstride()) {
    int64_t i = o - o_lo, ok = o + 1;
    okey[i] = ok;
    cust[i] = tqp_o_custkey(seed, sf, ok);
    date[i] = tqp_o_orderdate_days(seed, ok) * TQP_NS_PER_DAY;
    prio[i] = 0;
  }
}

template <int W, bool PART>
__global__ void k_str_maxlen(uint64_t seed, int64_t n, unsigned int* out) {
  unsigned int m = 1;
  uint8_t buf[W];
  for (int64_t i = gtid(); i < n; i += gstride()) {
    int len = PART ? tqp_p_type(seed, i, buf) : tqp_c_mktsegment(seed, i, buf);
    m = max(m, static_cast<unsigned int>(len));
  }
  atomicMax(out, m);
}

template <int W, bool PART>
__global__ void k_gen_strkey(uint64_t seed, int64_t lo, int64_t hi, int m, int64_t* __restrict__ key,
                             uint8_t* __restrict__ str) {
  uint8_t buf[W];
  for (int64_t i = lo + gtid(); i < hi; i += gstride()) {
    int64_t r = i - lo;
    key[r] = i + 1;
    if (PART) tqp_p_type(seed, i, buf);
    else tqp_c_mktsegment(seed, i, buf);
    for (int j = 0; j < m; ++j) str[r * m + j] = buf[j];
  }
}

}  // namespace

// Builds one shard of a generated table.
Table gen_table(Ctx& c, const std::string& name, double sf, uint64_t seed, int shard, int nshards) {
  if (nshards < 1 || shard < 0 || shard >= nshards) throw Error(TQP_ERR_ARG, "bad shard");
  Table t;
  if (name == "lineitem" || name == "orders") {
    int64_t L = tqp_lineitem_rows(sf);
    int64_t nmax = L / 4 + static_cast<int64_t>(4 * std::sqrt(static_cast<double>(L))) + 128;
    Tensor offs;
    int64_t n_orders = 0;
    while (true) {
      Tensor lines = c.alloc(TQP_I64, nmax, 1);
      k_order_lines<<<c.grid_for(nmax, 256), 256, 0, c.stream>>>(seed, nmax, lines.ptr<int64_t>());
      c.count_launch();
      int64_t ovf;
      offs = k::prefix_sum_raw(c, lines, &ovf);
      int64_t last = read_scalar<int64_t>(c, offs, nmax - 1) + read_scalar<int64_t>(c, lines, nmax - 1);
      if (last >= L) break;
      nmax = nmax * 3 / 2;
    }
    // n_orders = number of orders whose first line < L; shard bounds
    std::vector<int64_t> targets = {L};
    for (int s = 0; s <= nshards; ++s) targets.push_back(L * s / nshards);
    Tensor d_t = upload(c, TQP_I64, static_cast<int64_t>(targets.size()), 1, targets.data());
    Tensor d_o = c.alloc(TQP_I64, static_cast<int64_t>(targets.size()), 1);
    k_lower_bounds<<<1, 32, 0, c.stream>>>(offs.ptr<int64_t>(), nmax, d_t.ptr<int64_t>(),
                                           static_cast<int64_t>(targets.size()), d_o.ptr<int64_t>());
    c.count_launch();
    std::vector<int64_t> ob(targets.size());
    download(c, d_o, ob.data());
    n_orders = ob[0];
    int64_t o_lo = ob[1 + shard], o_hi = ob[2 + shard];
    if (shard == nshards - 1) o_hi = n_orders;
    if (o_hi > n_orders) o_hi = n_orders;
    if (o_lo > o_hi) o_lo = o_hi;
    if (name == "orders") {
      int64_t n = o_hi - o_lo;
      Tensor okey = c.alloc(TQP_I64, n, 1), cust = c.alloc(TQP_I64, n, 1), date = c.alloc(TQP_I64, n, 1),
             prio = c.alloc(TQP_I64, n, 1);
      if (n) {
        k_gen_orders<<<c.grid_for(n, 256), 256, 0, c.stream>>>(seed, sf, o_lo, o_hi, okey.ptr<int64_t>(),
                                                               cust.ptr<int64_t>(), date.ptr<int64_t>(),
                                                               prio.ptr<int64_t>());
        c.count_launch();
      }
      t.cols = {{"o_orderkey", TQP_LT_INT64, okey},
                {"o_custkey", TQP_LT_INT64, cust},
                {"o_orderdate", TQP_LT_DATE, date},
                {"o_shippriority", TQP_LT_INT64, prio}};
      t.rows = n;
    } else {
      int64_t row_lo = o_lo < n_orders ? read_scalar<int64_t>(c, offs, o_lo) : L;
      int64_t row_hi = o_hi < n_orders ? read_scalar<int64_t>(c, offs, o_hi) : L;
      int64_t n = row_hi - row_lo;
      Tensor okey = c.alloc(TQP_I64, n, 1), pkey = c.alloc(TQP_I64, n, 1), qty = c.alloc(TQP_I64, n, 1),
             price = c.alloc(TQP_F64, n, 1), disc = c.alloc(TQP_F64, n, 1), tax = c.alloc(TQP_F64, n, 1),
             rflag = c.alloc(TQP_STR8, n, 1), lstatus = c.alloc(TQP_STR8, n, 1), ship = c.alloc(TQP_I64, n, 1);
      LineitemCols lc{okey.ptr<int64_t>(), pkey.ptr<int64_t>(),  qty.ptr<int64_t>(),
                      ship.ptr<int64_t>(), price.ptr<double>(),  disc.ptr<double>(),
                      tax.ptr<double>(),   rflag.ptr<uint8_t>(), lstatus.ptr<uint8_t>()};
      if (o_hi > o_lo) {
        k_gen_lineitem<<<c.grid_for(o_hi - o_lo, 256), 256, 0, c.stream>>>(seed, sf, offs.ptr<int64_t>(), o_lo, o_hi,
                                                                           L, row_lo, lc);
        c.count_launch();
      }
      t.cols = {{"l_orderkey", TQP_LT_INT64, okey},     {"l_partkey", TQP_LT_INT64, pkey},
                {"l_quantity", TQP_LT_INT64, qty},      {"l_extendedprice", TQP_LT_FLOAT64, price},
                {"l_discount", TQP_LT_FLOAT64, disc},   {"l_tax", TQP_LT_FLOAT64, tax},
                {"l_returnflag", TQP_LT_UTF8, rflag},   {"l_linestatus", TQP_LT_UTF8, lstatus},
                {"l_shipdate", TQP_LT_DATE, ship}};
      t.rows = n;
    }
  } else if (name == "part" || name == "customer") {
    bool part = name == "part";
    int64_t N = part ? tqp_part_rows(sf) : tqp_customer_rows(sf);
    int64_t lo = N * shard / nshards, hi = N * (shard + 1) / nshards;
    auto mbuf = c.alloc_bytes(4);
    unsigned int one = 1;
    TQP_CUDA(cudaMemcpyAsync(mbuf->ptr, &one, 4, cudaMemcpyHostToDevice, c.stream));
    if (N) {
      if (part) k_str_maxlen<TQP_P_TYPE_WIDTH, true><<<c.grid_for(N, 256), 256, 0, c.stream>>>(seed, N, static_cast<unsigned*>(mbuf->ptr));
      else k_str_maxlen<TQP_C_SEG_WIDTH, false><<<c.grid_for(N, 256), 256, 0, c.stream>>>(seed, N, static_cast<unsigned*>(mbuf->ptr));
      c.count_launch();
    }
    unsigned int m = 1;
    TQP_CUDA(cudaMemcpyAsync(&m, mbuf->ptr, 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    int64_t n = hi - lo;
    Tensor key = c.alloc(TQP_I64, n, 1), str = c.alloc(TQP_STR8, n, m);
    if (n) {
      if (part) k_gen_strkey<TQP_P_TYPE_WIDTH, true><<<c.grid_for(n, 256), 256, 0, c.stream>>>(seed, lo, hi, m, key.ptr<int64_t>(), str.ptr<uint8_t>());
      else k_gen_strkey<TQP_C_SEG_WIDTH, false><<<c.grid_for(n, 256), 256, 0, c.stream>>>(seed, lo, hi, m, key.ptr<int64_t>(), str.ptr<uint8_t>());
      c.count_launch();
    }
    if (part) t.cols = {{"p_partkey", TQP_LT_INT64, key}, {"p_type", TQP_LT_UTF8, str}};
    else t.cols = {{"c_custkey", TQP_LT_INT64, key}, {"c_mktsegment", TQP_LT_UTF8, str}};
    t.rows = n;
  } else {
    throw Error(TQP_ERR_ARG, "unknown generated table '" + name + "'");
  }
  c.sync();
  return t;
}

}  // namespace tqp
