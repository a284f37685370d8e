// Builds the TPC-H-shaped tables of include/tqp_gen.h as reference
// EncodedTables through the reference's public API (Tensor::from_vector,
// tensor.hpp:53-57; Tensor::from_matrix; EncodedTable ctor, columnar.hpp:44).
// Test infrastructure: feeds the reference CPU executor the exact bytes the
// GPU path generates on device.
#pragma once

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "tensql/columnar.hpp"
#include "tensql/exec/interpreter.hpp"
#include "tensql/plan.hpp"
#include "tqp_gen.h"

namespace tqp_oracle {

using namespace tensql;

inline TableSchema lineitem_schema() {
  return {{"l_orderkey", LogicalType::Int64},   {"l_partkey", LogicalType::Int64},
          {"l_quantity", LogicalType::Int64},   {"l_extendedprice", LogicalType::Float64},
          {"l_discount", LogicalType::Float64}, {"l_tax", LogicalType::Float64},
          {"l_returnflag", LogicalType::Utf8},  {"l_linestatus", LogicalType::Utf8},
          {"l_shipdate", LogicalType::Date}};
}
inline TableSchema orders_schema() {
  return {{"o_orderkey", LogicalType::Int64},
          {"o_custkey", LogicalType::Int64},
          {"o_orderdate", LogicalType::Date},
          {"o_shippriority", LogicalType::Int64}};
}
inline TableSchema customer_schema() {
  return {{"c_custkey", LogicalType::Int64}, {"c_mktsegment", LogicalType::Utf8}};
}
inline TableSchema part_schema() {
  return {{"p_partkey", LogicalType::Int64}, {"p_type", LogicalType::Utf8}};
}

inline Catalog tpch_catalog() {
  Catalog c;
  c.add_table("lineitem", lineitem_schema());
  c.add_table("orders", orders_schema());
  c.add_table("customer", customer_schema());
  c.add_table("part", part_schema());
  return c;
}

// Order line offsets: offs[o] = first lineitem row of order o+1 (orderkey
// o+1); the last order is truncated so lineitem has exactly L rows.
inline std::vector<int64_t> order_offsets(uint64_t seed, double sf) {
  int64_t L = tqp_lineitem_rows(sf);
  std::vector<int64_t> offs;
  int64_t acc = 0;
  for (int64_t ok = 1; acc < L; ++ok) {
    offs.push_back(acc);
    acc += tqp_order_lines(seed, ok);
  }
  offs.push_back(L);
  return offs;  // size = n_orders + 1
}

template <typename F>
inline void parallel_ranges(int64_t n, F&& f) {
  int th = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> ts;
  for (int t = 0; t < th; ++t) {
    int64_t lo = n * t / th, hi = n * (t + 1) / th;
    ts.emplace_back([=, &f] { f(lo, hi); });
  }
  for (auto& t : ts) t.join();
}

inline TableSet tpch_tables(double sf, uint64_t seed) {
  auto offs = order_offsets(seed, sf);
  int64_t n_orders = static_cast<int64_t>(offs.size()) - 1;
  int64_t L = offs.back();

  std::vector<int64_t> okey(L), pkey(L), qty(L), ship(L);
  std::vector<double> price(L), disc(L), tax(L);
  std::vector<int32_t> rflag(L), lstatus(L);
  std::vector<int64_t> o_key(n_orders), o_cust(n_orders), o_date(n_orders), o_prio(n_orders, 0);
  parallel_ranges(n_orders, [&](int64_t lo, int64_t hi) {
    for (int64_t o = lo; o < hi; ++o) {
      int64_t ok = o + 1;
      int64_t od = tqp_o_orderdate_days(seed, ok);
      o_key[o] = ok;
      o_cust[o] = tqp_o_custkey(seed, sf, ok);
      o_date[o] = od * TQP_NS_PER_DAY;
      for (int64_t r = offs[o]; r < offs[o + 1]; ++r) {
        int64_t sd = tqp_l_shipdate_days(seed, r, od);
        okey[r] = ok;
        pkey[r] = tqp_l_partkey(seed, sf, r);
        qty[r] = tqp_l_quantity(seed, r);
        price[r] = tqp_l_extendedprice(seed, r);
        disc[r] = tqp_l_discount(seed, r);
        tax[r] = tqp_l_tax(seed, r);
        ship[r] = sd * TQP_NS_PER_DAY;
        rflag[r] = tqp_l_returnflag(seed, r, sd);
        lstatus[r] = tqp_l_linestatus(sd);
      }
    }
  });

  TableSet ts;
  ts["lineitem"] = EncodedTable({
      {"l_orderkey", LogicalType::Int64, Tensor::from_vector(std::move(okey))},
      {"l_partkey", LogicalType::Int64, Tensor::from_vector(std::move(pkey))},
      {"l_quantity", LogicalType::Int64, Tensor::from_vector(std::move(qty))},
      {"l_extendedprice", LogicalType::Float64, Tensor::from_vector(std::move(price))},
      {"l_discount", LogicalType::Float64, Tensor::from_vector(std::move(disc))},
      {"l_tax", LogicalType::Float64, Tensor::from_vector(std::move(tax))},
      {"l_returnflag", LogicalType::Utf8, Tensor::from_matrix(L, 1, std::move(rflag))},
      {"l_linestatus", LogicalType::Utf8, Tensor::from_matrix(L, 1, std::move(lstatus))},
      {"l_shipdate", LogicalType::Date, Tensor::from_vector(std::move(ship))},
  });
  ts["orders"] = EncodedTable({
      {"o_orderkey", LogicalType::Int64, Tensor::from_vector(std::move(o_key))},
      {"o_custkey", LogicalType::Int64, Tensor::from_vector(std::move(o_cust))},
      {"o_orderdate", LogicalType::Date, Tensor::from_vector(std::move(o_date))},
      {"o_shippriority", LogicalType::Int64, Tensor::from_vector(std::move(o_prio))},
  });

  // strings: width m = max byte length, as encode_string_rows does
  // (columnar.cpp:161-175)
  auto string_col = [&](int64_t n, int width, auto&& fill) {
    std::vector<uint8_t> bytes(static_cast<size_t>(n) * width);
    std::vector<int> lens(n);
    parallel_ranges(n, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) lens[i] = fill(i, bytes.data() + i * width);
    });
    int m = 1;
    for (int l : lens) m = std::max(m, l);
    std::vector<int32_t> data(static_cast<size_t>(n) * m);
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < m; ++j) data[i * m + j] = bytes[i * width + j];
    return Tensor::from_matrix(n, m, std::move(data));
  };

  int64_t NP = tqp_part_rows(sf), NC = tqp_customer_rows(sf);
  std::vector<int64_t> p_key(NP), c_key(NC);
  for (int64_t i = 0; i < NP; ++i) p_key[i] = i + 1;
  for (int64_t i = 0; i < NC; ++i) c_key[i] = i + 1;
  ts["part"] = EncodedTable({
      {"p_partkey", LogicalType::Int64, Tensor::from_vector(std::move(p_key))},
      {"p_type", LogicalType::Utf8,
       string_col(NP, TQP_P_TYPE_WIDTH, [&](int64_t i, uint8_t* o) { return tqp_p_type(seed, i, o); })},
  });
  ts["customer"] = EncodedTable({
      {"c_custkey", LogicalType::Int64, Tensor::from_vector(std::move(c_key))},
      {"c_mktsegment", LogicalType::Utf8,
       string_col(NC, TQP_C_SEG_WIDTH, [&](int64_t i, uint8_t* o) { return tqp_c_mktsegment(seed, i, o); })},
  });
  return ts;
}

}  // namespace tqp_oracle
