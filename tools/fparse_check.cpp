// Holds the CSV field parsers (paper_2209_04579_b200/csrc/fparse.cuh, the
// same code the device kernels run) to the reference's own parsers, byte for
// byte, on random and edge-case fields:
//   float64 / int64  std::from_chars (what CsvColumnBuilder::parse calls,
//                    columnar.cpp:398-412), value bits and accept/reject
//   date             tensql::encode_date (columnar.cpp:128-148) from the
//                    reference library, value and accept/reject
// Test infrastructure (links oracle/_ref/libtensql.a); run by
// tests/test_csv.py.   fparse_check [count] [seed]
#include <charconv>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "fparse.cuh"
#include "tensql/columnar.hpp"

using namespace tqp::fp;

static int failures = 0;

static void check_f64(const std::string& s) {
  double ref = 0;
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), ref);
  const bool ref_ok = ec == std::errc() && p == s.data() + s.size();
  uint64_t rb;
  std::memcpy(&rb, &ref, 8);
  uint64_t got = 0;
  const int r = parse_f64(reinterpret_cast<const unsigned char*>(s.data()), static_cast<int>(s.size()), got);
  const bool ok = r == 0;
  if (ok != ref_ok || (ok && got != rb)) {
    if (failures++ < 30)
      std::printf("f64 MISMATCH '%s': ref %s %016llx, got r=%d %016llx\n", s.c_str(), ref_ok ? "ok" : "err",
                  static_cast<unsigned long long>(rb), r, static_cast<unsigned long long>(got));
  }
}

static void check_i64(const std::string& s) {
  long long ref = 0;
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), ref);
  const bool ref_ok = ec == std::errc() && p == s.data() + s.size();
  int64_t got = 0;
  const bool ok = parse_i64(reinterpret_cast<const unsigned char*>(s.data()), static_cast<int>(s.size()), got) == 0;
  if (ok != ref_ok || (ok && got != ref)) {
    if (failures++ < 30) std::printf("i64 MISMATCH '%s'\n", s.c_str());
  }
}

static void check_date(const std::string& s) {
  int64_t ref = 0;
  bool ref_ok = true;
  try {
    ref = tensql::encode_date(s);
  } catch (const std::exception&) {
    ref_ok = false;
  }
  int64_t got = 0;
  int y, m, d;
  const bool ok = parse_date(reinterpret_cast<const unsigned char*>(s.data()), static_cast<int>(s.size()), got, y, m, d) == 0;
  if (ok != ref_ok || (ok && got != ref)) {
    if (failures++ < 30) std::printf("date MISMATCH '%s': ref %d, got %d\n", s.c_str(), ref_ok, ok);
  }
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 300000;
  std::mt19937_64 r(argc > 2 ? std::atoll(argv[2]) : 7);
  auto pick = [&](int k) { return static_cast<int>(r() % static_cast<uint64_t>(k)); };
  const std::vector<std::string> edges = {
      "0", "-0", "0.0", "1", "-1", "1.", ".5", ".", "-", "+1", "1e", "1e+", "1e5", "1E-5", "1.5e", "e5", "inf", "-inf",
      "INF", "Infinity", "infinit", "nan", "NaN", "-nan", "nan()", "nan(123)", "nan(a_b9)", "nan(-)", "nan(", "1e400",
      "-1e400", "1e-400", "4.9e-324", "2.4703282292062327e-324", "2.4703282292062328e-324", "5e-324", "3e-324",
      "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308", "2.2250738585072011e-308",
      "2.2250738585072014e-308", "9007199254740993", "9007199254740992.5", "1e23", "8.98846567431158e307",
      "123456789012345678901234567890", "0.1e-5", "-.5e-3", "0e999", "0.0e-500", "-0e400", "00000e5",
      "0e-99999999999", "1e-99999999999", "1e99999999999", "1e400x", "0x1p3", "1_0", " 1", "1 ", "00012",
      "0.000000000000000000000000000000000000001e-300", "9223372036854775807", "9223372036854775808",
      "-9223372036854775808", "-9223372036854775809", "18446744073709551616", "007",
      "2.225073858507201136057409796709131975934819546351645648023426109724822222021076945516529523908135087914149158913039621106870086438694594645527657207407820621743379988141063267329253552286881372149012981122451451889849057222307285255133155755015914397476397983411801999323962548289017107081850690630666655994938275772572015763062690663332647565300009245888316433037779791869612049497390377829704905051080609940730262937128958950003583799967207254304360284078895771796150945516748243471030702609144621572289880258182545180325707018860872113128079512233426288368622321503775666622503982534335974568884423900265498198385487948292206894721689831099698365846814022854243330660339850886445804001034933970427567186443383770486037861622771738545623065874679014086723327636718751234567890123456789e-308",
      "1.00000000000000011102230246251565404236316680908203125", "1.00000000000000011102230246251565404236316680908203124",
      "1.00000000000000011102230246251565404236316680908203126", "0.30000000000000004440892098500626161694526672363281250",
      "7.4109846876186981626485318930233205854758970392148714663837852375101326090531312779794975454245398856969484704316857659638998506553390969459816219401617281718945106978546710679176872575177347315553307795408549809608457500958111373034747658096871009590975442271004757307809711118935784838675653998783503015228055934046593739791790738723868299395818481660169122019456499931289798411362062484498678713572180352209017023903285791732520220528974020802906854021606612375549983402671300035812486479041385743401875520901590172592547146296175134159774938718574737870961645638908718119841271673056017045493004705269590165763776884908267986972573366521765567941072508764337560846003984904972149117463085539556354188641513168478436313080237596295773983001708984375e-318",
  };
  for (const auto& s : edges) {
    check_f64(s);
    check_i64(s);
  }
  for (long i = 0; i < n; ++i) {
    std::string s;
    const int kind = pick(10);
    if (kind < 4) {  // decimals of many shapes
      if (pick(4) == 0) s += '-';
      const int id = pick(25);
      for (int k = 0; k < id; ++k) s += static_cast<char>('0' + pick(10));
      if (pick(3)) {
        s += '.';
        const int fd = pick(kind == 0 ? 40 : 20);
        for (int k = 0; k < fd; ++k) s += static_cast<char>('0' + pick(10));
      }
      if (pick(2)) {
        s += "eE"[pick(2)];
        if (pick(2)) s += "+-"[pick(2)];
        s += std::to_string(pick(kind == 1 ? 400 : 30));
      }
    } else if (kind < 7) {  // random doubles printed exactly / nearly
      double v;
      uint64_t b = r();
      std::memcpy(&v, &b, 8);
      char buf[64];
      const int prec = pick(20);
      std::snprintf(buf, sizeof buf, pick(2) ? "%.*e" : "%.*g", prec, v);
      s = buf;
    } else if (kind < 8) {  // money-shaped
      char buf[64];
      std::snprintf(buf, sizeof buf, "%ld.%02d", static_cast<long>(r() % 10000000), pick(100));
      s = buf;
    } else if (kind < 9) {  // near-halfway decimals with many digits
      double v;
      uint64_t b = (r() & 0x7FEFFFFFFFFFFFFFULL);
      std::memcpy(&v, &b, 8);
      char buf[128];
      std::snprintf(buf, sizeof buf, "%.25e", v);
      s = buf;
      // perturb a late digit
      size_t pe = s.find('e');
      if (pe != std::string::npos && pe > 20) s[pe - 1 - pick(5)] = static_cast<char>('0' + pick(10));
    } else {  // random bytes from the number alphabet
      const char* al = "0123456789.-+eEinfatyINF()_ x";
      const int len = 1 + pick(12);
      for (int k = 0; k < len; ++k) s += al[pick(29)];
    }
    check_f64(s);
    check_i64(s);
  }
  // dates
  const std::vector<std::string> dedges = {"1970-01-01", "1992-02-29", "1993-02-29", "2000-02-29", "1900-02-29",
                                           "2262-04-11", "2262-04-12", "1677-09-21", "1677-09-22", "1677-09-20",
                                           "-001-02-03", "0000-01-01", "9999-12-31", "1995-13-01", "1995-00-10",
                                           "1995-01-00", "1995-1-010", "1995/01/01", "19950101", "1995-01-01 ",
                                           "1995-0-101", "+995-01-01", "1995--1-01", "1995-01--1", "----------"};
  for (const auto& s : dedges) check_date(s);
  for (long i = 0; i < n / 10; ++i) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%04d-%02d-%02d", 1600 + pick(800), pick(14), pick(33));
    std::string s = buf;
    if (pick(20) == 0) s[pick(10)] = "-0123456789x"[pick(12)];
    check_date(s);
  }
  std::printf("fparse_check: %ld random + %zu edge fields, %d mismatch(es)\n", n, edges.size(), failures);
  return failures ? 1 : 0;
}
