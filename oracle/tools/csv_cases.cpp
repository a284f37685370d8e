// Golden CSV cases for the device loader: every case is
// parsed by the UNMODIFIED reference (tensql::parse_csv_text,
// columnar.cpp:453-519) and written with its table or its exact error text.
// Test infrastructure (links oracle/_ref/libtensql.a); run by
// oracle/make_golden.sh:   csv_cases OUT.json
#include <fstream>
#include <iostream>
#include <random>
#include <string>
#include <vector>

#include <chrono>
#include <cstdio>

#include "dump.hpp"
#include "tpch_tables.hpp"

using namespace tqp_oracle;

namespace {

json cases = json::array();

std::string hex(const std::string& s) {
  static const char* d = "0123456789abcdef";
  std::string o;
  for (unsigned char c : s) {
    o += d[c >> 4];
    o += d[c & 15];
  }
  return o;
}

void add(const std::string& name, const std::string& text, const TableSchema& schema, char delim = ',') {
  json c;
  c["name"] = name;
  c["text_hex"] = hex(text);
  c["delimiter"] = std::string(1, delim);
  json sch = json::array();
  for (const auto& col : schema) sch.push_back({col.name, logical_type_name(col.type)});
  c["schema"] = sch;
  try {
    EncodedTable t = parse_csv_text(text, schema, delim, "t.csv");
    c["result"] = table_to_json(t);
  } catch (const std::exception& e) {
    c["error"] = e.what();
  }
  cases.push_back(c);
}

const TableSchema kAll = {{"i", LogicalType::Int64}, {"f", LogicalType::Float64}, {"d", LogicalType::Date},
                          {"s", LogicalType::Utf8},  {"b", LogicalType::Bool}};

void fixed_cases() {
  const std::string H = "i,f,d,s,b\n";
  add("basic", H + "1,2.5,1995-03-15,hello,true\n-7,-0.0,1970-01-01,w\xc3\xa9,0\n", kAll);
  add("no trailing newline", H + "1,2.5,1995-03-15,x,1", kAll);
  add("two trailing newlines", H + "1,2.5,1995-03-15,x,1\n\n", kAll);
  add("crlf", "i,f,d,s,b\r\n1,2.5,1995-03-15,x,1\r\n2,3,1995-03-16,yy,false\r\n", kAll);
  add("crlf blank tail", "i,f,d,s,b\r\n1,2.5,1995-03-15,x,1\r\n\r\n", kAll);
  add("header only", H, kAll);
  add("header only no newline", "i,f,d,s,b", kAll);
  add("header case", "I,F,D,S,B\n1,1,1995-01-01,a,1\n", kAll);
  add("pipe delimiter", "i|f|d|s|b\n1|1e5|1995-01-01|a,b|true\n", kAll, '|');
  add("tab delimiter", "i\tf\td\ts\tb\n1\t.5\t1995-01-01\ta b\tfalse\n", kAll, '\t');
  add("floats", std::string("f\n") + "1.\n.5\n1e5\n1E-5\n-.5e-3\ninf\n-inf\nINF\nInfinity\nnan\nNaN\n-nan\nnan(123)\n"
          "00012\n4.9e-324\n2.4703282292062328e-324\n1.7976931348623157e308\n1.7976931348623158e308\n"
          "9007199254740993\n1e23\n123456789012345678901234567890\n0e999\n-0e400\n0.1\n0.2\n0.30000000000000004\n"
          "1.00000000000000011102230246251565404236316680908203125\n"
          "1.00000000000000011102230246251565404236316680908203126\n",
      {{"f", LogicalType::Float64}});
  add("ints", std::string("i\n") + "0\n-0\n007\n9223372036854775807\n-9223372036854775808\n", {{"i", LogicalType::Int64}});
  add("dates", std::string("d\n") + "1970-01-01\n2000-02-29\n-001-02-03\n0000-01-01\n1677-09-22\n2262-04-11\n",
      {{"d", LogicalType::Date}});
  add("utf8", std::string("s\n") + "a\nhello world\n\xe2\x82\xac\n\xf0\x9f\x98\x80\nx,y\n", {{"s", LogicalType::Utf8}}, '|');
  // errors
  add("empty text", "", kAll);
  add("empty schema", "i\n1\n", {});
  add("header count", "i,f\n1,2\n", kAll);
  add("header name", "i,f,d,q,b\n", kAll);
  add("field count", H + "1,2.5,1995-03-15,x,1\n1,2.5,1995-03-15,x\n", kAll);
  add("field count extra", H + "1,2.5,1995-03-15,x,1,9\n", kAll);
  add("blank middle line", H + "1,2.5,1995-03-15,x,1\n\n1,2.5,1995-03-15,x,1\n", kAll);
  add("empty int", H + ",2.5,1995-03-15,x,1\n", kAll);
  add("empty utf8", H + "1,2.5,1995-03-15,,1\n", kAll);
  for (const char* v : {"+1", "1 ", " 1", "1.0", "9223372036854775808", "-9223372036854775809", "-", "0x10", "1e3"})
    add(std::string("bad int ") + v, std::string("i\n") + v + "\n", {{"i", LogicalType::Int64}});
  for (const char* v : {"+1", ".", "-", "1e", "1e+", "1.5e", "e5", "1e400", "-1e400", "1e-400", "2.4703282292062327e-324",
                        "1.7976931348623159e308", "0x1p3", "1_0", "infinit", "nan(", "nan(-)", "1 ",
                        "2.4703282292062327208828439643411068618252990130716238221279284125033775363510437593264991818081799618989828234772285886546332835517796989819938739800539093906315035659515570226392290858392449105184435931802849936536152500319370457678249219365623669863658480757001585769269903706311928279558551332927834338409351978015531246597263579574622766465272827220056374006485499977096599470454020828166226237857393450736339007967761930577506740176324673600968951340535537458516661134223766678604162159680461914467291840300530057530849048765391711386591646239524912623653881879636239373280423891018672348497668235089863388587925628302755995657524455507255189313690836254779186948667994968324049705821028513185451396213837722826145437693412532098591327667236328125e-324"})
    add(std::string("bad float ") + std::string(v).substr(0, 24), std::string("f\n1\n") + v + "\n", {{"f", LogicalType::Float64}});
  for (const char* v : {"1995-13-01", "1995-00-10", "1995-02-30", "1993-02-29", "1900-02-29", "1995/01/01", "19950101",
                        "1995-1-010", "+995-01-01", "1995--1-01", "1995-01--1", "2262-04-12", "1677-09-21",
                        "9999-12-31", "1995-01-01 "})
    add(std::string("bad date ") + v, std::string("d\n") + v + "\n", {{"d", LogicalType::Date}});
  for (const char* v : {"yes", "True", "2", "t", "false "}) add(std::string("bad bool ") + v, std::string("b\n") + v + "\n", {{"b", LogicalType::Bool}});
  add("bad utf8 overlong", std::string("s\n") + "\xc0\x80" + "\n", {{"s", LogicalType::Utf8}});
  add("bad utf8 truncated", std::string("s\n") + "ab\xe2\x82" + "\n", {{"s", LogicalType::Utf8}});
  add("bad utf8 lead", std::string("s\n") + "\xf8\x88\x80\x80\x80" + "\n", {{"s", LogicalType::Utf8}});
  add("bad utf8 nul", std::string("s\n") + std::string("a\0b", 3) + "\n", {{"s", LogicalType::Utf8}});
  add("first error wins (row order)", H + "1,2.5,1995-03-15,x,1\n1,bad,1995-03-15,x,1\nzz,2.5,1995-03-15,x,1\n", kAll);
  add("first error wins (field order)", H + "1,2.5,1995-03-15,x,1\n1,bad,1995-02-30,,maybe\n", kAll);
  add("count before fields", H + "zz,2.5,1995-03-15,x,1\n1,2,3\n", kAll);
}

void random_cases(int n, uint64_t seed) {
  std::mt19937_64 r(seed);
  auto pick = [&](int k) { return static_cast<int>(r() % static_cast<uint64_t>(k)); };
  for (int c = 0; c < n; ++c) {
    const char delims[] = {',', '|', ';', '\t'};
    const char delim = delims[pick(4)];
    std::string text = "i";
    text += delim;
    text += "f";
    text += delim;
    text += "d";
    text += delim;
    text += "s";
    text += delim;
    text += "b\n";
    const int rows = pick(250);
    const char* words[] = {"A", "N", "R", "PROMO BRUSHED", "x", "long value with spaces", "\xc3\xa9t\xc3\xa9", "0"};
    for (int i = 0; i < rows; ++i) {
      char buf[256];
      double v;
      uint64_t bits = r();
      std::memcpy(&v, &bits, 8);
      std::string f;
      switch (pick(5)) {
        case 0: snprintf(buf, sizeof buf, "%.2f", static_cast<double>(pick(10000000)) / 100.0); f = buf; break;
        case 1: snprintf(buf, sizeof buf, "%.17g", v); f = buf; break;
        case 2: snprintf(buf, sizeof buf, "%.*e", pick(22), v); f = buf; break;
        case 3: snprintf(buf, sizeof buf, "%d.%d", pick(100000), pick(100)); f = buf; break;
        default: snprintf(buf, sizeof buf, "%.25g", static_cast<double>(pick(1000000)) / 7.0); f = buf; break;
      }
      if (f.find("nan") != std::string::npos || f.find("inf") != std::string::npos) f = "0.5";
      snprintf(buf, sizeof buf, "%lld", static_cast<long long>(r()) >> pick(60));
      text += buf;
      text += delim;
      text += f;
      text += delim;
      snprintf(buf, sizeof buf, "%04d-%02d-%02d", 1970 + pick(60), 1 + pick(12), 1 + pick(28));
      text += buf;
      text += delim;
      text += words[pick(8)];
      text += delim;
      text += pick(2) ? (pick(2) ? "true" : "1") : (pick(2) ? "false" : "0");
      text += pick(8) ? "\n" : "\r\n";
    }
    add("random " + std::to_string(c), text, kAll, delim);
  }
}

}  // namespace

// lineitem of the shared generator as CSV text (two-decimal money, ISO dates)
int write_lineitem(double sf, const char* path) {
  TableSet ts = tpch_tables(sf, 7);
  const EncodedTable& t = ts.at("lineitem");
  auto rows = decode_table(t);
  FILE* f = std::fopen(path, "wb");
  if (!f) return 1;
  for (size_t c = 0; c < t.columns().size(); ++c) std::fprintf(f, "%s%s", c ? "," : "", t.columns()[c].name.c_str());
  std::fputc('\n', f);
  for (const auto& r : rows) {
    for (size_t c = 0; c < r.size(); ++c) {
      if (c) std::fputc(',', f);
      const LogicalType lt = t.columns()[c].logical;
      if (lt == LogicalType::Float64) std::fprintf(f, "%.2f", std::get<double>(r[c]));
      else std::fputs(cell_to_text(r[c], lt).c_str(), f);
    }
    std::fputc('\n', f);
  }
  std::fclose(f);
  return 0;
}

// the reference's load_csv on a file (CPU baseline of the loader)
int time_reference(const char* path, int reps) {
  double best = 1e30;
  int64_t rows = 0;
  for (int i = 0; i < reps; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    EncodedTable t = load_csv(path, lineitem_schema(), ',');
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    best = ms < best ? ms : best;
    rows = t.row_count();
  }
  std::printf("{\"rows\": %lld, \"ms\": %.3f}\n", static_cast<long long>(rows), best);
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 4 && std::string(argv[1]) == "lineitem") return write_lineitem(std::stod(argv[2]), argv[3]);
  if (argc >= 3 && std::string(argv[1]) == "time") return time_reference(argv[2], argc > 3 ? std::stoi(argv[3]) : 1);
  if (argc < 2) {
    std::cerr << "usage: csv_cases OUT.json | csv_cases lineitem SF OUT.csv | csv_cases time FILE.csv [reps]\n";
    return 2;
  }
  fixed_cases();
  random_cases(16, 11);
  std::ofstream(argv[1]) << json({{"generator", "oracle/tools/csv_cases.cpp (reference parse_csv_text)"}, {"cases", cases}}).dump()
                         << "\n";
  return 0;
}
