// rnla_cli -- command-line drop-in for the hot-path subcommands of the
// reference CLI (tools/randnla_cli.cpp:127-445): sketch, lsr, ksvd, spsd,
// nystrom, cur (kernel mode). Same flags, one JSON RunReport per line on stdout
// (schemas/run_report.schema.json: command, seed, parameters, metrics,
// status, elapsed_ms, message; keys sorted like the reference's std::map),
// a human summary on stderr, exit codes 0 ok / 2 flagged / 1 error. Matrix
// files: Matrix Market (.mtx/.mm, array or coordinate, general or symmetric)
// or CSV (src/io.cpp:47-230). Every computation runs through the C ABI
// (include/rnla.h) via the C++ facade; the other reference subcommands
// (verify, dense cur, apps, bench) are outside the B200 build and report an error.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "randnla_b200/randnla.hpp"

using namespace randnla_b200;

namespace {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ matrix I/O
std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

bool to_double(const std::string& t, double& v) {
  const char* e = t.data() + t.size();
  auto r = std::from_chars(t.data(), e, v);
  return r.ec == std::errc() && r.ptr == e;
}
bool to_long(const std::string& t, long& v) {
  const char* e = t.data() + t.size();
  auto r = std::from_chars(t.data(), e, v);
  return r.ec == std::errc() && r.ptr == e;
}

std::vector<std::string> tokens(const std::string& line) {
  std::vector<std::string> out;
  std::istringstream in(line);
  for (std::string t; in >> t;) out.push_back(t);
  return out;
}

[[noreturn]] void bad(const std::string& path, long line, const std::string& what) {
  throw ParseError(path + ":" + std::to_string(line) + ": " + what);
}

bool is_matrix_market(const std::string& path) {
  const auto dot = path.find_last_of('.');
  const std::string ext = dot == std::string::npos ? "" : lower(path.substr(dot + 1));
  return ext == "mtx" || ext == "mm";
}

DenseMatrix read_mm(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError(path + ": cannot open file");
  std::string line;
  long no = 0;
  if (!std::getline(in, line)) bad(path, 1, "empty file");
  ++no;
  const auto h = tokens(lower(line));
  if (h.size() < 4 || h[0] != "%%matrixmarket" || h[1] != "matrix") bad(path, no, "not a Matrix Market header");
  if (h[2] != "array" && h[2] != "coordinate") bad(path, no, "unsupported layout '" + h[2] + "'");
  if (h[3] != "real" && h[3] != "integer") bad(path, no, "unsupported field '" + h[3] + "'");
  const bool sym = h.size() > 4 && h[4] == "symmetric";
  if (h.size() > 4 && h[4] != "general" && !sym) bad(path, no, "unsupported symmetry '" + h[4] + "'");
  const bool coord = h[2] == "coordinate";
  std::vector<std::string> sz;
  while (std::getline(in, line)) {
    ++no;
    if (!line.empty() && line[0] == '%') continue;
    sz = tokens(line);
    if (!sz.empty()) break;
  }
  long rows = 0, cols = 0, nnz = 0;
  if (sz.size() != (coord ? 3u : 2u) || !to_long(sz[0], rows) || !to_long(sz[1], cols) || rows < 0 || cols < 0 ||
      (coord && (!to_long(sz[2], nnz) || nnz < 0)))
    bad(path, no, "malformed size line");
  DenseMatrix m(rows, cols);
  long count = 0;
  const long total = coord ? nnz : (sym ? rows * (rows + 1) / 2 : rows * cols);
  long i = 0, j = 0;
  while (std::getline(in, line)) {
    ++no;
    if (!line.empty() && line[0] == '%') continue;
    const auto t = tokens(line);
    if (t.empty()) continue;
    if (coord) {
      long r = 0, c = 0;
      double v = 0.0;
      if (t.size() != 3) bad(path, no, "expected 'i j value'");
      if (!to_long(t[0], r) || !to_long(t[1], c) || !to_double(t[2], v)) bad(path, no, "malformed entry");
      if (r < 1 || r > rows || c < 1 || c > cols) bad(path, no, "entry index out of bounds");
      m(r - 1, c - 1) = v;
      if (sym) m(c - 1, r - 1) = v;
      ++count;
    } else {
      for (const auto& tok : t) {
        double v = 0.0;
        if (!to_double(tok, v)) bad(path, no, "malformed value");
        if (count >= total) bad(path, no, "more values than declared");
        m(i, j) = v;
        if (sym) m(j, i) = v;
        if (++i == rows) {
          ++j;
          i = sym ? j : 0;
        }
        ++count;
      }
    }
  }
  if (count != total)
    bad(path, no, (coord ? "entry count mismatch: header says " : "value count mismatch: expected ") +
                      std::to_string(total) + ", file has " + std::to_string(count));
  return m;
}

DenseMatrix read_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError(path + ": cannot open file");
  std::vector<std::vector<double>> rows;
  std::string line;
  long no = 0;
  while (std::getline(in, line)) {
    ++no;
    if (line.empty()) continue;
    std::vector<double> row;
    std::stringstream cells(line);
    for (std::string cell; std::getline(cells, cell, ',');) {
      const auto a = cell.find_first_not_of(" \t\r"), b = cell.find_last_not_of(" \t\r");
      if (a == std::string::npos) bad(path, no, "empty cell");
      cell = cell.substr(a, b - a + 1);
      double v = 0.0;
      if (!to_double(cell, v)) bad(path, no, "malformed value '" + cell + "'");
      row.push_back(v);
    }
    if (row.empty()) bad(path, no, "empty row");
    if (!rows.empty() && row.size() != rows.front().size())
      bad(path, no,
          "row has " + std::to_string(row.size()) + " cells, expected " + std::to_string(rows.front().size()));
    rows.push_back(std::move(row));
  }
  if (rows.empty()) throw ParseError(path + ": empty file");
  DenseMatrix m((Index)rows.size(), (Index)rows.front().size());
  for (size_t r = 0; r < rows.size(); ++r)
    for (size_t c = 0; c < rows[r].size(); ++c) m((Index)r, (Index)c) = rows[r][c];
  return m;
}

DenseMatrix load_matrix(const std::string& path) { return is_matrix_market(path) ? read_mm(path) : read_csv(path); }

std::string num17(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
  return std::string(buf, r.ptr);
}

void save_matrix(const DenseMatrix& m, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error(path + ": cannot open for writing");
  if (is_matrix_market(path)) {
    out << "%%MatrixMarket matrix array real general\n" << m.rows() << ' ' << m.cols() << '\n';
    for (Index j = 0; j < m.cols(); ++j)
      for (Index i = 0; i < m.rows(); ++i) out << num17(m(i, j)) << '\n';
  } else {
    for (Index i = 0; i < m.rows(); ++i) {
      for (Index j = 0; j < m.cols(); ++j) out << (j ? "," : "") << num17(m(i, j));
      out << '\n';
    }
  }
  if (!out) throw std::runtime_error(path + ": write failure");
}

// -------------------------------------------------------------- small host math
double fro(const DenseMatrix& a) {
  double s = 0.0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) s += a(i, j) * a(i, j);
  return std::sqrt(s);
}
DenseMatrix mul(const DenseMatrix& a, const DenseMatrix& b, bool ta = false, bool tb = false) {
  const Index m = ta ? a.cols() : a.rows(), k = ta ? a.rows() : a.cols(), n = tb ? b.rows() : b.cols();
  DenseMatrix c(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index p = 0; p < k; ++p) {
      const double bv = tb ? b(j, p) : b(p, j);
      if (bv == 0.0) continue;
      for (Index i = 0; i < m; ++i) c(i, j) += (ta ? a(p, i) : a(i, p)) * bv;
    }
  return c;
}
DenseMatrix minus(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix c(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) c(i, j) = a(i, j) - b(i, j);
  return c;
}

// ------------------------------------------------------------------ RunReport
struct Report {
  std::string command;
  std::uint64_t seed = 0;
  std::map<std::string, std::string> parameters;
  std::map<std::string, double> metrics;
  std::string status = "ok";
  std::string message;
};

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    if (c == '"') o += "\\\"";
    else if (c == '\\') o += "\\\\";
    else if (c == '\n') o += "\\n";
    else if (c == '\t') o += "\\t";
    else if (c == '\r') o += "\\r";
    else if (c < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else o += (char)c;
  }
  return o + "\"";
}

// Shortest round-trip decimal, with ".0" on integral values (as JSON libraries print doubles).
std::string jnum(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".en") == std::string::npos) s += ".0";
  return s;
}

void emit(const Report& rep, double ms) {
  for (const auto& kv : rep.metrics)
    if (!std::isfinite(kv.second)) throw std::runtime_error("non-finite metric '" + kv.first + "'");
  std::string j = "{\"command\":" + jstr(rep.command) + ",\"seed\":" + std::to_string(rep.seed) + ",\"parameters\":{";
  bool first = true;
  for (const auto& kv : rep.parameters) {
    j += (first ? "" : ",") + jstr(kv.first) + ":" + jstr(kv.second);
    first = false;
  }
  j += "},\"metrics\":{";
  first = true;
  for (const auto& kv : rep.metrics) {
    j += (first ? "" : ",") + jstr(kv.first) + ":" + jnum(kv.second);
    first = false;
  }
  j += "},\"status\":" + jstr(rep.status) + ",\"elapsed_ms\":" + jnum(ms);
  if (!rep.message.empty()) j += ",\"message\":" + jstr(rep.message);
  std::cout << j << "}\n";
  std::cerr << rep.command << " [" << rep.status << "]";
  for (const auto& kv : rep.metrics) std::cerr << ' ' << kv.first << '=' << kv.second;
  if (!rep.message.empty()) std::cerr << " -- " << rep.message;
  std::cerr << '\n';
}

// ------------------------------------------------------------------ options
struct Args {
  std::map<std::string, std::string> kv;
  std::vector<std::string> flags;
  bool has(const std::string& k) const { return kv.count(k) > 0; }
  bool flag(const std::string& k) const { return std::find(flags.begin(), flags.end(), k) != flags.end(); }
  std::string str(const std::string& k, const std::string& d = "") const { return has(k) ? kv.at(k) : d; }
  long long i64(const std::string& k, long long d = 0) const { return has(k) ? std::stoll(kv.at(k)) : d; }
  std::uint64_t u64(const std::string& k) const { return has(k) ? std::stoull(kv.at(k)) : 0; }
  double f64(const std::string& k, double d) const { return has(k) ? std::stod(kv.at(k)) : d; }
};

struct UsageError : std::runtime_error {
  int code;
  UsageError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};

Args parse(int argc, char** argv, const std::vector<std::string>& valued, const std::vector<std::string>& flag_names,
           const std::vector<std::string>& required, const std::vector<std::string>& files) {
  Args a;
  for (int i = 2; i < argc; ++i) {
    std::string t = argv[i], v;
    const auto eq = t.find('=');
    if (eq != std::string::npos) {
      v = t.substr(eq + 1);
      t = t.substr(0, eq);
    }
    if (std::find(flag_names.begin(), flag_names.end(), t) != flag_names.end()) {
      a.flags.push_back(t);
      continue;
    }
    if (std::find(valued.begin(), valued.end(), t) == valued.end())
      throw UsageError("The following argument was not expected: " + t, 109);
    if (eq == std::string::npos) {
      if (i + 1 >= argc) throw UsageError(t + " requires an argument", 107);
      v = argv[++i];
    }
    a.kv[t] = v;
  }
  for (const auto& r : required)
    if (!a.has(r)) throw UsageError(r + " is required", 106);
  for (const auto& f : files)
    if (a.has(f) && !std::ifstream(a.str(f)).good())
      throw UsageError(f + ": File does not exist: " + a.str(f), 105);
  return a;
}

SketchKind kind_of(const std::string& name) {
  if (name == "gaussian") return SketchKind::kGaussian;
  if (name == "srht") return SketchKind::kSrht;
  if (name == "count") return SketchKind::kCountSketch;
  if (name == "uniform") return SketchKind::kUniformColumns;
  if (name == "leverage") return SketchKind::kLeverageColumns;
  if (name == "landmark") return SketchKind::kLandmarkColumns;
  throw UsageError("--method: unknown sketch kind '" + name + "'", 105);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "A subcommand is required (sketch, lsr, ksvd, spsd, nystrom)\n";
    return 106;
  }
  const std::string cmd = argv[1];
  Report rep;
  rep.command = cmd;
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  try {
    try {
      if (cmd == "sketch") {
        Args a = parse(argc, argv, {"--input", "--method", "--s", "--s-cs", "--seed", "--output"}, {},
                       {"--input", "--s", "--seed"}, {"--input"});
        rep.seed = a.u64("--seed");
        const std::string method = a.str("--method", "gaussian");
        const Index s = a.i64("--s");
        rep.parameters = {{"input", a.str("--input")}, {"method", method}, {"s", std::to_string(s)}};
        const DenseMatrix m = load_matrix(a.str("--input"));
        SketchSpec spec;
        if (method == "combined") {
          const Index s_cs = a.i64("--s-cs") > 0 ? a.i64("--s-cs") : 4 * s;
          spec = SketchSpec::combined(s_cs, SketchSpec::gaussian(s, derive_seed(rep.seed, 1)), rep.seed);
        } else {
          spec.kind = kind_of(method);
          spec.s = s;
          spec.seed = rep.seed;
        }
        const DenseMatrix c = apply_sketch(m, spec);
        if (a.has("--output")) save_matrix(c, a.str("--output"));
        rep.metrics["input_fro"] = fro(m);
        rep.metrics["sketch_fro"] = fro(c);
        rep.metrics["sketch_cols"] = (double)c.cols();
      } else if (cmd == "lsr") {
        Args a = parse(argc, argv,
                       {"--method", "--input", "--rhs", "--sketch", "--sketch-size", "--eps", "--tol", "--maxit",
                        "--seed", "--output"},
                       {"--cg"}, {"--input", "--rhs"}, {"--input", "--rhs"});
        const std::string method = a.str("--method", "exact");
        if ((method == "sketched" || method == "preconditioned") && !a.has("--seed"))
          throw std::invalid_argument("--seed is required for --method " + method);
        rep.seed = a.u64("--seed");
        rep.parameters = {{"method", method}, {"input", a.str("--input")}, {"rhs", a.str("--rhs")}};
        const DenseMatrix A = load_matrix(a.str("--input"));
        const DenseMatrix B = load_matrix(a.str("--rhs"));
        if (B.cols() != 1) throw std::invalid_argument("--rhs must be a single column");
        Vector b(B.rows());
        for (Index i = 0; i < B.rows(); ++i) b(i) = B(i, 0);
        const std::string sk = a.str("--sketch", "count");
        LsrSolution sol;
        if (method == "exact") {
          sol = lsr_exact(A, b);
        } else if (method == "cg") {
          sol = lsr_cg(A, b, a.f64("--tol", 1e-10), (int)a.i64("--maxit", 1000));
        } else if (method == "sketched") {
          SketchSpec spec;
          spec.kind = kind_of(sk);
          spec.s = a.i64("--sketch-size") > 0 ? a.i64("--sketch-size") : 20 * A.cols();
          spec.seed = rep.seed;
          sol = lsr_sketched(A, b, spec);
        } else if (method == "preconditioned") {
          PreconditionedOptions po;
          po.sketch_size = a.i64("--sketch-size");
          po.use_cg = a.flag("--cg");
          po.sketch_kind = kind_of(sk);
          sol = lsr_preconditioned(A, b, a.f64("--eps", 1e-8), rep.seed, po);
        } else {
          throw std::invalid_argument("unknown method '" + method + "'");
        }
        if (a.has("--output")) {
          DenseMatrix x(sol.x.size(), 1);
          for (Index i = 0; i < sol.x.size(); ++i) x(i, 0) = sol.x(i);
          save_matrix(x, a.str("--output"));
        }
        rep.metrics["objective"] = sol.objective;
        rep.metrics["iterations"] = sol.iterations;
        if (sol.kappa_estimate) rep.metrics["kappa"] = *sol.kappa_estimate;
        if (sol.flagged) rep.status = "flagged";
      } else if (cmd == "ksvd") {
        Args a = parse(argc, argv, {"--method", "--input", "--k", "--s", "--p", "--p-cs", "--q", "--seed", "--output"},
                       {}, {"--input", "--k", "--seed"}, {"--input"});
        rep.seed = a.u64("--seed");
        const std::string method = a.str("--method", "prototype");
        const Index k = a.i64("--k");
        rep.parameters = {{"method", method}, {"input", a.str("--input")}, {"k", std::to_string(k)}};
        const DenseMatrix m = load_matrix(a.str("--input"));
        const Index s = a.i64("--s") > 0 ? a.i64("--s") : 4 * k;
        KsvdOptions ko;
        ko.evaluate_error = true;
        KsvdResult r;
        if (method == "prototype") {
          r = prototype_ksvd(m, k, s, rep.seed, nullptr, ko);
        } else if (method == "faster") {
          const Index p = a.i64("--p") > 0 ? a.i64("--p") : 4 * s;
          const Index p_cs = a.i64("--p-cs") > 0 ? a.i64("--p-cs") : 4 * p;
          r = faster_ksvd(m, k, s, p_cs, p, rep.seed, ko);
        } else if (method == "lanczos") {
          throw std::runtime_error("block_lanczos_ksvd is not part of the B200 hot path (DESIGN.md section 6)");
        } else {
          throw std::invalid_argument("unknown method '" + method + "'");
        }
        if (a.has("--output")) {
          DenseMatrix us(r.factors.U.rows(), r.factors.U.cols());
          for (Index j = 0; j < us.cols(); ++j)
            for (Index i = 0; i < us.rows(); ++i) us(i, j) = r.factors.U(i, j) * r.factors.singular_values(j);
          save_matrix(mul(us, r.factors.V, false, true), a.str("--output"));
        }
        rep.metrics["error_fro"] = *r.error_fro;
        rep.metrics["passes"] = r.passes_over_a;
        rep.metrics["top_sv"] = r.factors.singular_values(0);
      } else if (cmd == "spsd") {
        Args a = parse(argc, argv, {"--data", "--sigma", "--s", "--p", "--method", "--seed"}, {},
                       {"--data", "--sigma", "--s", "--seed"}, {"--data"});
        rep.seed = a.u64("--seed");
        const std::string method = a.str("--method", "faster");
        const Index s = a.i64("--s");
        const double sigma = a.f64("--sigma", 1.0);
        rep.parameters = {{"data", a.str("--data")}, {"method", method}, {"s", std::to_string(s)}};
        const DenseMatrix x = load_matrix(a.str("--data"));
        const DenseMatrix kernel = rbf_kernel(x, x, sigma);
        DenseMatrix Q, Z;
        bool flagged = false;
        if (method == "prototype") {
          // spsd_prototype (src/spsd.cpp:117-129): Q = U of the count sketch of K, Z = Q'KQ
          if (!(s >= 1 && s <= kernel.cols())) throw std::invalid_argument("spsd_prototype: s > n");
          Q = condensed_svd(apply_sketch(kernel, SketchSpec::count_sketch(s, rep.seed))).U;
          Z = mul(mul(Q, kernel, true, false), Q);
          for (Index i = 0; i < Z.rows(); ++i)
            for (Index j = i + 1; j < Z.cols(); ++j) Z(i, j) = Z(j, i) = 0.5 * (Z(i, j) + Z(j, i));
        } else if (method == "faster") {
          const Index p = std::min<Index>(a.i64("--p") > 0 ? a.i64("--p") : 4 * s, x.rows());
          const SpsdSketch sk = spsd_faster(x, KernelSpec{sigma}, s, p, rep.seed);
          Q = sk.Q;
          Z = sk.Z;
          flagged = sk.flagged;
          const double sec = (double)sk.secondary.size();
          rep.metrics["kernel_entries"] = (double)x.rows() * (double)s + sec * sec;
        } else {
          throw std::invalid_argument("unknown method '" + method + "'");
        }
        rep.metrics["error_rel"] = fro(minus(kernel, mul(mul(Q, Z), Q, false, true))) / fro(kernel);
        if (flagged) rep.status = "flagged";
      } else if (cmd == "nystrom") {
        Args a = parse(argc, argv, {"--data", "--sigma", "--l", "--k", "--seed"}, {}, {"--data", "--sigma", "--seed"},
                       {"--data"});
        rep.seed = a.u64("--seed");
        const Index l = a.i64("--l", 100);
        rep.parameters = {{"data", a.str("--data")}, {"l", std::to_string(l)}};
        const DenseMatrix x = load_matrix(a.str("--data"));
        const double sigma = a.f64("--sigma", 1.0);
        const NystromFactor f = nystrom(x, KernelSpec{sigma}, std::min<Index>(l, x.rows()), rep.seed, a.i64("--k"));
        const DenseMatrix kernel = rbf_kernel(x, x, sigma);
        rep.metrics["error_rel"] = fro(minus(kernel, mul(f.L, f.L, false, true))) / fro(kernel);
        rep.metrics["rank"] = (double)f.L.cols();
      } else if (cmd == "cur") {
        Args a = parse(argc, argv,
                       {"--input", "--train", "--test", "--sigma", "--method", "--c", "--r", "--p-c", "--p-r", "--seed",
                        "--output"},
                       {"--leverage"}, {"--c", "--r", "--seed"}, {"--input", "--train", "--test"});
        rep.seed = a.u64("--seed");
        const Index c = a.i64("--c", 10), r = a.i64("--r", 10);
        rep.parameters = {{"method", a.str("--method", "faster")}, {"c", std::to_string(c)}, {"r", std::to_string(r)}};
        if (a.has("--input")) {
          rep.parameters["input"] = a.str("--input");
          throw std::runtime_error("dense CUR (cur_prototype / cur_faster) is not part of the B200 hot path; "
                                   "use --train/--test (cur_faster_kernel)");
        }
        if (!a.has("--train") || !a.has("--test"))
          throw std::invalid_argument("provide --input (dense) or --train and --test (kernel)");
        rep.parameters["train"] = a.str("--train");
        rep.parameters["test"] = a.str("--test");
        const DenseMatrix xtrain = load_matrix(a.str("--train")), xtest = load_matrix(a.str("--test"));
        const CurFactors f = cur_faster_kernel(xtest, xtrain, a.f64("--sigma", 1.0), c, r, rep.seed);
        if (a.has("--output")) save_matrix(mul(f.C, mul(f.U, f.R)), a.str("--output"));
        rep.metrics["entries_visited"] = (double)f.entries_visited;
        rep.metrics["core_rows"] = (double)f.U.rows();
        rep.metrics["core_cols"] = (double)f.U.cols();
        if (f.flagged) rep.status = "flagged";
      } else {
        throw UsageError("The following argument was not expected: " + cmd +
                             " (this build provides sketch, lsr, ksvd, spsd, nystrom, cur)",
                         109);
      }
    } catch (const UsageError&) {
      throw;
    } catch (const std::exception& e) {
      rep.status = "error";
      rep.message = e.what();
      rep.metrics.clear();
    }
    emit(rep, elapsed());
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return e.code;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
  return rep.status == "ok" ? 0 : (rep.status == "flagged" ? 2 : 1);
}
