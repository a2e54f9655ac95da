// Host-only checks of include/nlem_b200_io.hpp against the behaviour the reference documents
// for its file formats (proj/include/nlem/pgm.hpp, point_set_io.hpp, csv.hpp) and restates
// its unit-test expectations (proj/tests/unit/test_pgm.cpp, test_point_set_io.cpp,
// test_csv.cpp).  No GPU: run on the CPU suite.  Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <string>

#include "nlem_b200_io.hpp"

static int failures = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
      ++failures;                                                         \
    }                                                                     \
  } while (0)

template <class F>
static bool throws_parse(F&& f, std::size_t* offset = nullptr, std::string* what = nullptr) {
  try {
    f();
  } catch (const nlem::ParseError& e) {
    if (offset) *offset = e.byte_offset();
    if (what) *what = e.what();
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::string bytes_of(const std::string& header, std::initializer_list<int> raster) {
  std::string s = header;
  for (int b : raster) s.push_back(static_cast<char>(b));
  return s;
}

int main() {
  // ---- PGM decode
  {
    const nlem::Image a = nlem::decode_pgm("P2\n# comment\n4   1\n#x\n255\n10 64\t128\n255\n");
    CHECK(a.rows() == 1 && a.cols() == 4);
    CHECK(a(0, 0) == 10 && a(0, 1) == 64 && a(0, 2) == 128 && a(0, 3) == 255);
    const nlem::Image b = nlem::decode_pgm(bytes_of("P5\n4 1\n255\n", {10, 64, 128, 255}));
    CHECK(b.cols() == 4 && b(0, 0) == 10 && b(0, 3) == 255);
    const nlem::Image w = nlem::decode_pgm(bytes_of("P5\n2 1\n1000\n", {0x01, 0x00, 0x00, 0xFF}));
    CHECK(w(0, 0) == 256 && w(0, 1) == 255);  // two bytes, big-endian
    const nlem::Image h = nlem::decode_pgm("P2\n2 1\n1000\n999 0\n");
    CHECK(h(0, 0) == 999 && h(0, 1) == 0);
  }
  // ---- PGM encode: round half away from zero, clamp to [0, 255]
  {
    nlem::Image img(1, 5);
    const float v[5] = {-3.2f, 254.7f, 99.5f, 12.0f, 300.0f};
    for (int i = 0; i < 5; ++i) img(0, i) = v[i];
    const nlem::Image back = nlem::decode_pgm(nlem::encode_pgm(img, nlem::PgmFormat::P2));
    CHECK(back(0, 0) == 0 && back(0, 1) == 255 && back(0, 2) == 100 && back(0, 3) == 12 &&
          back(0, 4) == 255);
  }
  // ---- integral images survive both encodings; re-encoding reproduces the bytes
  {
    std::mt19937_64 rng(101);
    nlem::Image img(9, 13);
    for (auto& x : img.data_) x = static_cast<float>(rng() % 256);
    for (auto f : {nlem::PgmFormat::P2, nlem::PgmFormat::P5}) {
      const std::string s = nlem::encode_pgm(img, f);
      const nlem::Image back = nlem::decode_pgm(s);
      CHECK(back.rows() == 9 && back.cols() == 13 && back.data_ == img.data_);
      CHECK(nlem::encode_pgm(back, f) == s);
    }
    nlem::Image wide(3, 40, 255.0f);
    std::istringstream lines(nlem::encode_pgm(wide, nlem::PgmFormat::P2));
    std::string line;
    while (std::getline(lines, line)) CHECK(line.size() <= 70);
  }
  // ---- every corruption of the magic is rejected
  {
    const std::string bases[2] = {"P2\n4 1\n255\n10 64 128 255\n",
                                  bytes_of("P5\n4 1\n255\n", {10, 64, 128, 255})};
    int accepted = 0;
    for (const auto& base : bases)
      for (int pos = 0; pos < 2; ++pos)
        for (int b = 0; b < 256; ++b) {
          std::string m = base;
          if (m[pos] == static_cast<char>(b)) continue;
          m[pos] = static_cast<char>(b);
          if (!throws_parse([&] { nlem::decode_pgm(m); })) ++accepted;
        }
    CHECK(accepted == 0);
  }
  // ---- malformed headers / rasters name the offending byte
  {
    std::size_t off = 0;
    CHECK(throws_parse([] { nlem::decode_pgm(bytes_of("P5\n4 1\n255\n", {10, 64, 128})); }));
    const std::string t = "P2\n2 1\n100\n50 101\n";
    CHECK(throws_parse([&] { nlem::decode_pgm(t); }, &off) && off == t.find("101"));
    const std::string p = bytes_of("P5\n2 1\n200\n", {10, 201});
    CHECK(throws_parse([&] { nlem::decode_pgm(p); }, &off) && off == p.size() - 1);
    CHECK(throws_parse([] { nlem::decode_pgm("P2\n"); }));
    CHECK(throws_parse([] { nlem::decode_pgm("P2\n4\n"); }));
    CHECK(throws_parse([] { nlem::decode_pgm("P2\n0 1\n255\n"); }));
    CHECK(throws_parse([] { nlem::decode_pgm("P2\n1 0\n255\n"); }));
    CHECK(throws_parse([] { nlem::decode_pgm("P2\n1 1\n0\n5\n"); }));
    CHECK(throws_parse([] { nlem::decode_pgm("P2\n1 1\n65536\n5\n"); }));
    CHECK(!throws_parse([] { nlem::decode_pgm("P2\n1 1\n255\n7\n \t\n"); }));
    const std::string tr = "P2\n1 1\n255\n7\n8\n";
    CHECK(throws_parse([&] { nlem::decode_pgm(tr); }, &off) && off == tr.size() - 2);
    std::string what;
    CHECK(throws_parse([] { nlem::decode_pgm("P2\n1 1\n255\n7 x"); }, nullptr, &what) &&
          what.find("byte offset") != std::string::npos);
  }
  // ---- point sets
  {
    const nlem::PointSet ps = nlem::decode_point_set("2 3\n0 0.5 -1 1\n2.25 3 4 0.125\n");
    CHECK(ps.size() == 2 && ps.dim() == 3);
    CHECK(ps.points[0] == 0.0f && ps.points[1] == 0.5f && ps.points[2] == -1.0f && ps.weights[0] == 1.0f);
    CHECK(ps.points[3] == 2.25f && ps.points[4] == 3.0f && ps.points[5] == 4.0f && ps.weights[1] == 0.125f);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<float> u(-1e3f, 1e3f);
    nlem::PointSet r;
    r.d = 5;
    for (int i = 0; i < 35; ++i) r.points.push_back(u(rng));
    for (int i = 0; i < 7; ++i) r.weights.push_back(std::abs(u(rng)) + 0.5f);
    const nlem::PointSet back = nlem::decode_point_set(nlem::encode_point_set(r));
    CHECK(back.points == r.points && back.weights == r.weights && back.d == 5);
    std::size_t off = 99;
    std::string what;
    CHECK(throws_parse([] { nlem::decode_point_set("x 3\n"); }, &off, &what) && off == 0 &&
          what.find("point count") != std::string::npos);
    CHECK(throws_parse([] { nlem::decode_point_set(" 2 y\n"); }, &off, &what) && off == 3 &&
          what.find("dimension") != std::string::npos);
    const std::string bad = "1 2\n1 abc 1\n";
    CHECK(throws_parse([&] { nlem::decode_point_set(bad); }, &off) && off == bad.find("abc"));
    const std::string extra = "1 1\n3 1\nextra\n";
    CHECK(throws_parse([&] { nlem::decode_point_set(extra); }, &off, &what) && off == extra.find("extra") &&
          what.find("trailing") != std::string::npos);
    CHECK(throws_parse([] { nlem::decode_point_set("0 2\n"); }));
    CHECK(throws_parse([] { nlem::decode_point_set("1 0\n"); }));
    CHECK(throws_parse([] { nlem::decode_point_set("1 1\n3 0\n"); }));    // no positive weight
    CHECK(throws_parse([] { nlem::decode_point_set("1 1\n3 -1\n"); }));   // negative weight
    CHECK(throws_parse([] { nlem::decode_point_set("1 1\n3\n"); }));      // truncated
    CHECK(throws_parse([] { nlem::read_point_set_file("/nonexistent/nlem_points.txt"); }, nullptr, &what) &&
          what.find("nlem_points.txt") != std::string::npos);
  }
  // ---- CSV grammars
  {
    CHECK(nlem::encode_trace_csv({}) == "iter,objective,primal_residual\n");
    nlem::TraceRecord rec;
    rec.iter = 1;
    rec.objective = 7.25f;
    CHECK(nlem::encode_trace_csv({rec}) == "iter,objective,primal_residual\n1,7.25,\n");
    rec.primal_residual = 0.5f;
    CHECK(nlem::encode_trace_csv({rec}) == "iter,objective,primal_residual\n1,7.25,0.5\n");
    CHECK(nlem::encode_psnr_csv({20.5, 21.0}) == "iter,psnr\n1,20.5\n2,21\n");
    nlem::BenchRow b;
    b.image = "ramp";
    b.sigma = 20;
    b.method = "admm";
    b.mean_psnr = 30.25;
    b.std_psnr = 0;
    b.repeats = 2;
    CHECK(nlem::encode_bench_csv({b}) == "image,sigma,method,mean_psnr,std_psnr,R\nramp,20,admm,30.25,0,2\n");
  }
  // ---- mirror index, psnr
  {
    CHECK(nlem::mirror_index(-1, 5) == 1 && nlem::mirror_index(5, 5) == 3 && nlem::mirror_index(-2, 1) == 0);
    nlem::Image a(2, 2, 10.0f), b(2, 2, 10.0f);
    CHECK(std::isinf(nlem::psnr(a, b)));
    b(0, 0) = 12.0f;  // mse = 1
    CHECK(std::abs(nlem::psnr(a, b) - 10.0 * std::log10(255.0 * 255.0)) < 1e-12);
  }
  std::printf("%s (%d failed checks)\n", failures ? "FAILED" : "ok", failures);
  return failures;
}
