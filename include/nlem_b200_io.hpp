// nlem_b200_io.hpp — host-side file formats and helpers of the reference's front end, for the
// CLI (paper_1501_03879_b200/cli/nlem_main.cpp) and C++ users:
//   * PGM P2/P5 decode/encode             proj/include/nlem/pgm.hpp, proj/src/pgm.cpp
//   * text point sets ("n d", n lines)    proj/include/nlem/point_set_io.hpp, src/point_set_io.cpp
//   * trace / PSNR / bench CSV grammars   proj/include/nlem/csv.hpp, proj/src/csv.cpp
//   * PSNR against the 8-bit peak         proj/include/nlem/psnr.hpp:12-24
//   * Gaussian noise (forwarded to the C-ABI generator, noise.cpp:7-17)
//   * one pixel's patch stack on the host (patch.cpp:9-16, :27-38, :52-61, :63-88) and the
//     initial patch (nlem.cpp:13-18) — for per-pixel traces of the standalone solvers.
// Error behaviour follows the reference: ParseError(what, byte offset) for malformed content
// ("... (byte offset N)"), std::runtime_error for filesystem trouble, std::invalid_argument for
// invalid values.  Images are float here (the compute path is FP32); PGM samples are integers
// up to 65535, exactly representable.
#pragma once

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "nlem_b200.hpp"

namespace nlem {

class ParseError : public std::runtime_error {  // types.hpp:34-44
 public:
  ParseError(const std::string& what, std::size_t byte_offset)
      : std::runtime_error(what + " (byte offset " + std::to_string(byte_offset) + ")"),
        byte_offset_(byte_offset) {}
  std::size_t byte_offset() const { return byte_offset_; }

 private:
  std::size_t byte_offset_;
};

namespace io_detail {

inline std::string slurp(const std::string& path, bool parse_error_on_open) {
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    if (parse_error_on_open) throw ParseError("cannot open point-set file: " + path, 0);
    throw std::runtime_error("cannot open " + path + " for reading");
  }
  std::ostringstream buf;
  buf << in.rdbuf();
  if (in.bad()) throw std::runtime_error("failed reading " + path);
  return buf.str();
}

inline void save(const std::string& bytes, const std::string& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
  if (!out) throw std::runtime_error("failed writing " + path);
}

// "%.17g": the decimal form is injective over doubles (csv.cpp:13-17)
inline std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

}  // namespace io_detail

// ------------------------------------------------------------------------------------ PGM
enum class PgmFormat { P2, P5 };

// pgm.cpp: magic in the first two bytes, whitespace/'#'-comment separated header, maxval
// 1..65535, P5 raster one byte per sample (two, big-endian, above 255) after exactly one
// whitespace byte, nothing but whitespace after the raster.
inline Image decode_pgm(std::string_view b) {
  std::size_t pos = 0;
  auto skip = [&]() {
    while (pos < b.size()) {
      const unsigned char ch = static_cast<unsigned char>(b[pos]);
      if (std::isspace(ch)) {
        ++pos;
      } else if (ch == '#') {
        while (pos < b.size() && b[pos] != '\n') ++pos;
      } else {
        break;
      }
    }
  };
  auto uint_tok = [&](const char* what, long maxv) -> long {
    skip();
    const std::size_t start = pos;
    if (start >= b.size()) throw ParseError(std::string("missing ") + what, b.size());
    long v = 0;
    std::size_t digits = 0;
    while (pos < b.size() && std::isdigit(static_cast<unsigned char>(b[pos]))) {
      v = v * 10 + (b[pos] - '0');
      if (v > maxv) throw ParseError(std::string(what) + " out of range", start);
      ++pos;
      ++digits;
    }
    if (digits == 0) throw ParseError(std::string("malformed ") + what, start);
    return v;
  };
  auto byte = [&](const char* what) -> unsigned char {
    if (pos >= b.size()) throw ParseError(std::string("truncated ") + what, b.size());
    return static_cast<unsigned char>(b[pos++]);
  };
  if (b.size() < 2 || b[0] != 'P' || (b[1] != '2' && b[1] != '5'))
    throw ParseError("not a P2/P5 PGM file", 0);
  const bool binary = b[1] == '5';
  pos = 2;
  const long width = uint_tok("width", 1L << 30);
  const long height = uint_tok("height", 1L << 30);
  if (width < 1) throw ParseError("width must be positive", pos);
  if (height < 1) throw ParseError("height must be positive", pos);
  const long maxval = uint_tok("maxval", 65535);
  if (maxval < 1) throw ParseError("maxval must be positive", pos);
  Image img(height, width);
  if (binary) {
    const unsigned char sep = byte("raster");
    if (!std::isspace(sep)) throw ParseError("missing separator before binary raster", pos - 1);
    const bool wide = maxval > 255;
    for (long i = 0; i < height * width; ++i) {
      const std::size_t at = pos;
      long s = byte("raster");
      if (wide) s = s * 256 + byte("raster");
      if (s > maxval) throw ParseError("sample exceeds maxval", at);
      img.data_[i] = static_cast<float>(s);
    }
  } else {
    for (long i = 0; i < height * width; ++i) {
      skip();
      const std::size_t at = pos;
      const long s = uint_tok("sample", 65535);
      if (s > maxval) throw ParseError("sample exceeds maxval", at);
      img.data_[i] = static_cast<float>(s);
    }
  }
  skip();
  if (pos < b.size()) throw ParseError("trailing data after pixel samples", pos);
  return img;
}

// maxval 255; samples rounded half away from zero and clamped to [0, 255]; P2 lines carry 17
// samples (<= 70 characters).  Non-finite intensities are rejected (image.hpp:14-17).
inline std::string encode_pgm(const Image& img, PgmFormat fmt) {
  for (float v : img.data_)
    if (!std::isfinite(v)) throw std::invalid_argument("image intensities must be finite");
  if (img.rows() < 1 || img.cols() < 1) throw std::invalid_argument("image must be non-empty");
  auto q = [](float v) {
    const double r = std::round(static_cast<double>(v));
    return r < 0.0 ? 0 : (r > 255.0 ? 255 : static_cast<int>(r));
  };
  char hdr[64];
  std::snprintf(hdr, sizeof hdr, "%s\n%ld %ld\n255\n", fmt == PgmFormat::P2 ? "P2" : "P5",
                static_cast<long>(img.cols()), static_cast<long>(img.rows()));
  std::string out = hdr;
  if (fmt == PgmFormat::P5) {
    for (float v : img.data_) out.push_back(static_cast<char>(q(v)));
    return out;
  }
  int on_line = 0;
  for (float v : img.data_) {
    out += std::to_string(q(v));
    if (++on_line == 17) {
      out.push_back('\n');
      on_line = 0;
    } else {
      out.push_back(' ');
    }
  }
  if (on_line) out.push_back('\n');
  return out;
}

inline Image read_pgm(const std::string& path) { return decode_pgm(io_detail::slurp(path, false)); }
inline void write_pgm(const Image& img, const std::string& path, PgmFormat fmt) {
  io_detail::save(encode_pgm(img, fmt), path);
}

// ------------------------------------------------------------------------------ point sets
// types.hpp:58-68
inline void validate(const PointSet& ps) {
  if (ps.size() < 1) throw std::invalid_argument("point set must contain at least one point");
  if (static_cast<int64_t>(ps.weights.size()) != ps.size())
    throw std::invalid_argument("weight count does not match point count");
  for (float v : ps.points)
    if (!std::isfinite(v)) throw std::invalid_argument("point coordinates must be finite");
  bool pos = false;
  for (float w : ps.weights) {
    if (!std::isfinite(w) || w < 0.0f) throw std::invalid_argument("weights must be finite and nonnegative");
    pos |= w > 0.0f;
  }
  if (!pos) throw std::invalid_argument("at least one weight must be positive");
}

// point_set_io.cpp: "n d" then n lines of d coordinates and a weight, whitespace-separated
inline PointSet decode_point_set(const std::string& t) {
  std::size_t pos = 0;
  auto next = [&](std::string& tok, std::size_t& at) -> bool {
    while (pos < t.size() && std::isspace(static_cast<unsigned char>(t[pos]))) ++pos;
    if (pos >= t.size()) return false;
    at = pos;
    const std::size_t s = pos;
    while (pos < t.size() && !std::isspace(static_cast<unsigned char>(t[pos]))) ++pos;
    tok.assign(t, s, pos - s);
    return true;
  };
  auto int_tok = [&](const char* what) -> long long {
    std::string tok;
    std::size_t at = pos;
    if (!next(tok, at)) throw ParseError(std::string("unexpected end of input, expected ") + what, at);
    errno = 0;
    char* end = nullptr;
    const long long v = std::strtoll(tok.c_str(), &end, 10);
    if (errno != 0 || end == tok.c_str() || *end != '\0')
      throw ParseError(std::string("invalid integer for ") + what + ": '" + tok + "'", at);
    return v;
  };
  auto num_tok = [&](const char* what) -> double {
    std::string tok;
    std::size_t at = pos;
    if (!next(tok, at)) throw ParseError(std::string("unexpected end of input, expected ") + what, at);
    char* end = nullptr;
    const double v = std::strtod(tok.c_str(), &end);
    if (end == tok.c_str() || *end != '\0')
      throw ParseError(std::string("invalid number for ") + what + ": '" + tok + "'", at);
    return v;
  };
  const long long n = int_tok("point count n");
  const long long d = int_tok("dimension d");
  if (n < 1) throw ParseError("point count must be at least 1", 0);
  if (d < 1) throw ParseError("dimension must be at least 1", 0);
  PointSet ps;
  ps.d = d;
  ps.points.resize(static_cast<size_t>(n * d));
  ps.weights.resize(static_cast<size_t>(n));
  for (long long k = 0; k < n; ++k) {
    for (long long i = 0; i < d; ++i) ps.points[k * d + i] = static_cast<float>(num_tok("coordinate"));
    ps.weights[k] = static_cast<float>(num_tok("weight"));
  }
  std::string extra;
  std::size_t at = 0;
  if (next(extra, at)) throw ParseError("trailing data after last point", at);
  try {
    validate(ps);
  } catch (const std::invalid_argument& e) {
    throw ParseError(e.what(), 0);
  }
  return ps;
}

inline PointSet read_point_set_file(const std::string& path) {
  return decode_point_set(io_detail::slurp(path, true));
}

inline std::string encode_point_set(const PointSet& ps) {
  std::string out = std::to_string(ps.size()) + ' ' + std::to_string(ps.dim()) + '\n';
  for (int64_t k = 0; k < ps.size(); ++k) {
    for (int64_t i = 0; i < ps.dim(); ++i) out += io_detail::g17(ps.points[k * ps.dim() + i]) + ' ';
    out += io_detail::g17(ps.weights[k]) + '\n';
  }
  return out;
}

// ---------------------------------------------------------------------------------- CSVs
inline std::string encode_trace_csv(const std::vector<TraceRecord>& trace) {
  std::string out = "iter,objective,primal_residual\n";
  for (const auto& r : trace) {
    out += std::to_string(r.iter) + ',' + io_detail::g17(r.objective) + ',';
    if (!std::isnan(r.primal_residual)) out += io_detail::g17(r.primal_residual);
    out += '\n';
  }
  return out;
}

inline std::string encode_psnr_csv(const std::vector<double>& psnr_per_iter) {
  std::string out = "iter,psnr\n";
  for (size_t t = 0; t < psnr_per_iter.size(); ++t)
    out += std::to_string(t + 1) + ',' + io_detail::g17(psnr_per_iter[t]) + '\n';
  return out;
}

struct BenchRow {  // csv.hpp:24-31
  std::string image;
  double sigma = 0.0;
  std::string method;
  double mean_psnr = 0.0;
  double std_psnr = 0.0;
  int repeats = 0;
};

inline std::string encode_bench_csv(const std::vector<BenchRow>& rows) {
  std::string out = "image,sigma,method,mean_psnr,std_psnr,R\n";
  for (const auto& r : rows)
    out += r.image + ',' + io_detail::g17(r.sigma) + ',' + r.method + ',' + io_detail::g17(r.mean_psnr) +
           ',' + io_detail::g17(r.std_psnr) + ',' + std::to_string(r.repeats) + '\n';
  return out;
}

// --------------------------------------------------------------------------- quality, noise
inline double mse(const Image& ref, const Image& test) {  // psnr.hpp:12-16
  if (ref.rows() != test.rows() || ref.cols() != test.cols())
    throw std::invalid_argument("mse requires images of equal dimensions");
  double s = 0.0;
  for (size_t i = 0; i < ref.data_.size(); ++i) {
    const double e = static_cast<double>(ref.data_[i]) - static_cast<double>(test.data_[i]);
    s += e * e;
  }
  return s / static_cast<double>(ref.data_.size());
}

inline double psnr(const Image& ref, const Image& test) {  // psnr.hpp:20-24
  const double err = mse(ref, test);
  if (err == 0.0) return std::numeric_limits<double>::infinity();
  return 10.0 * std::log10(255.0 * 255.0 / err);
}

// noise.cpp:7-17 (unclipped), through the C-ABI generator
inline Image add_gaussian_noise(const Image& clean, double sigma, uint64_t seed) {
  if (!(sigma >= 0.0)) throw std::invalid_argument("noise sigma must be nonnegative");
  std::vector<double> c(clean.data_.begin(), clean.data_.end()), o(c.size());
  nlem_add_gaussian_noise(c.data(), static_cast<int64_t>(c.size()), sigma, seed, o.data());
  Image out(clean.rows(), clean.cols());
  for (size_t i = 0; i < o.size(); ++i) out.data_[i] = static_cast<float>(o[i]);
  return out;
}

}  // namespace nlem
