// aggmg_cli.cpp — the reference command line (proj/tools/aggmg_main.cpp) over the B200 drop-in:
// `generate`, `solve` and `bench` with the reference's options, defaults, console output, JSON
// report / run manifest and exit codes (0 ok, 2 no convergence, 3 input error).  The reference
// parses with CLI11 and writes with nlohmann::json (vendored there, absent here): this file has
// its own small option parser, JSON writer and manifest reader, with the same field names and
// order.  Built by `make` as build/aggmg.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "aggmg/aggmg.hpp"

namespace {

using Clock = std::chrono::steady_clock;
constexpr int kExitOk = 0;
constexpr int kExitNoConvergence = 2;
constexpr int kExitInputError = 3;

double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

// ---- a minimal ordered JSON value (what the report and the manifest need) ---------------------
struct Json {
  enum Kind { kNull, kBool, kInt, kNum, kStr, kArr, kObj } kind = kNull;
  bool b = false;
  long long i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  Json() = default;
  Json(bool v) : kind(kBool), b(v) {}                       // NOLINT
  Json(int v) : kind(kInt), i(v) {}                         // NOLINT
  Json(long long v) : kind(kInt), i(v) {}                   // NOLINT
  Json(long v) : kind(kInt), i(v) {}                        // NOLINT
  Json(unsigned long long v) : kind(kInt), i(static_cast<long long>(v)) {}  // NOLINT
  Json(unsigned long v) : kind(kInt), i(static_cast<long long>(v)) {}       // NOLINT
  Json(double v) : kind(kNum), d(v) {}                      // NOLINT
  Json(const char* v) : kind(kStr), s(v) {}                 // NOLINT
  Json(std::string v) : kind(kStr), s(std::move(v)) {}      // NOLINT
  Json(const std::vector<double>& v) : kind(kArr) {         // NOLINT
    for (double x : v) arr.emplace_back(x);
  }
  static Json object() {
    Json j;
    j.kind = kObj;
    return j;
  }
  static Json array() {
    Json j;
    j.kind = kArr;
    return j;
  }
  Json& operator[](const std::string& k) {
    if (kind == kNull) kind = kObj;
    for (auto& kv : obj)
      if (kv.first == k) return kv.second;
    obj.emplace_back(k, Json());
    return obj.back().second;
  }
  const Json& at(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw aggmg::Error("manifest: missing key '" + k + "'");
  }
  void push_back(Json v) {
    kind = kArr;
    arr.push_back(std::move(v));
  }

  static void esc(std::ostream& o, const std::string& v) {
    o << '"';
    for (char c : v) {
      if (c == '"' || c == '\\') o << '\\' << c;
      else if (c == '\n') o << "\\n";
      else if (static_cast<unsigned char>(c) < 0x20) o << "\\u" << std::hex << std::setw(4) << std::setfill('0') << int(c) << std::dec;
      else o << c;
    }
    o << '"';
  }
  static void num(std::ostream& o, double v) {
    if (!std::isfinite(v)) {
      o << "null";
      return;
    }
    char buf[32];
    auto r = std::to_chars(buf, buf + sizeof buf, v);  // shortest round-trip form
    std::string t(buf, r.ptr);
    if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
    o << t;
  }
  void dump(std::ostream& o, int indent, int depth) const {
    const std::string pad = indent > 0 ? std::string(static_cast<size_t>(indent * (depth + 1)), ' ') : "";
    const std::string pad0 = indent > 0 ? std::string(static_cast<size_t>(indent * depth), ' ') : "";
    const char* nl = indent > 0 ? "\n" : "";
    const char* colon = indent > 0 ? ": " : ":";
    switch (kind) {
      case kNull: o << "null"; break;
      case kBool: o << (b ? "true" : "false"); break;
      case kInt: o << i; break;
      case kNum: num(o, d); break;
      case kStr: esc(o, s); break;
      case kArr:
        if (arr.empty()) {
          o << "[]";
          break;
        }
        o << '[' << nl;
        for (size_t q = 0; q < arr.size(); ++q) {
          o << pad;
          arr[q].dump(o, indent, depth + 1);
          if (q + 1 < arr.size()) o << ',';
          o << nl;
        }
        o << pad0 << ']';
        break;
      case kObj:
        if (obj.empty()) {
          o << "{}";
          break;
        }
        o << '{' << nl;
        for (size_t q = 0; q < obj.size(); ++q) {
          o << pad;
          esc(o, obj[q].first);
          o << colon;
          obj[q].second.dump(o, indent, depth + 1);
          if (q + 1 < obj.size()) o << ',';
          o << nl;
        }
        o << pad0 << '}';
        break;
    }
  }
  std::string dump(int indent = -1) const {
    std::ostringstream o;
    dump(o, indent, 0);
    return o.str();
  }

  // parser (objects, arrays, strings, numbers, booleans, null)
  static Json parse(const std::string& text) {
    size_t p = 0;
    Json j = parse_value(text, p);
    skip(text, p);
    aggmg::require(p == text.size(), "manifest: trailing characters");
    return j;
  }
  static void skip(const std::string& t, size_t& p) {
    while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p]))) ++p;
  }
  static Json parse_value(const std::string& t, size_t& p) {
    skip(t, p);
    aggmg::require(p < t.size(), "manifest: unexpected end");
    const char c = t[p];
    if (c == '{') {
      Json j = object();
      ++p;
      skip(t, p);
      if (t[p] == '}') {
        ++p;
        return j;
      }
      while (true) {
        skip(t, p);
        const std::string k = parse_string(t, p);
        skip(t, p);
        aggmg::require(p < t.size() && t[p] == ':', "manifest: expected ':'");
        ++p;
        j.obj.emplace_back(k, parse_value(t, p));
        skip(t, p);
        if (t[p] == ',') { ++p; continue; }
        aggmg::require(t[p] == '}', "manifest: expected '}'");
        ++p;
        return j;
      }
    }
    if (c == '[') {
      Json j = array();
      ++p;
      skip(t, p);
      if (t[p] == ']') {
        ++p;
        return j;
      }
      while (true) {
        j.arr.push_back(parse_value(t, p));
        skip(t, p);
        if (t[p] == ',') { ++p; continue; }
        aggmg::require(t[p] == ']', "manifest: expected ']'");
        ++p;
        return j;
      }
    }
    if (c == '"') return Json(parse_string(t, p));
    if (t.compare(p, 4, "true") == 0) { p += 4; return Json(true); }
    if (t.compare(p, 5, "false") == 0) { p += 5; return Json(false); }
    if (t.compare(p, 4, "null") == 0) { p += 4; return Json(); }
    size_t e = p;
    while (e < t.size() && (std::isdigit(static_cast<unsigned char>(t[e])) || std::strchr("+-.eE", t[e]))) ++e;
    const std::string tok = t.substr(p, e - p);
    aggmg::require(!tok.empty(), "manifest: bad value");
    p = e;
    if (tok.find_first_of(".eE") == std::string::npos) return Json(std::stoll(tok));
    return Json(std::stod(tok));
  }
  static std::string parse_string(const std::string& t, size_t& p) {
    aggmg::require(p < t.size() && t[p] == '"', "manifest: expected a string");
    std::string out;
    for (++p; p < t.size() && t[p] != '"'; ++p) {
      if (t[p] == '\\' && p + 1 < t.size()) {
        ++p;
        out += t[p] == 'n' ? '\n' : t[p];
      } else {
        out += t[p];
      }
    }
    ++p;
    return out;
  }
  double num_value() const { return kind == kInt ? static_cast<double>(i) : d; }
  long long int_value() const { return kind == kInt ? i : static_cast<long long>(d); }
};

// aggmg_main.cpp:46-61
std::string file_hash(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  aggmg::require(in.good(), "cannot open '" + path + "' for hashing");
  std::uint64_t h = 1469598103934665603ULL;
  char buf[65536];
  while (in.read(buf, sizeof(buf)) || in.gcount() > 0) {
    for (std::streamsize i = 0; i < in.gcount(); ++i) {
      h ^= static_cast<unsigned char>(buf[i]);
      h *= 1099511628211ULL;
    }
  }
  std::ostringstream s;
  s << "fnv1a64:" << std::hex << std::setfill('0') << std::setw(16) << h;
  return s.str();
}

// aggmg_main.cpp:63-84: every solve setting with its default
struct SolveOptions {
  std::string matrix;
  std::string rhs;
  double tol = 1e-6;
  int max_iters = 200;
  int restart = 30;
  std::string solver = "fgmres";
  std::string cycle = "hybrid";
  int klevels = 2;
  std::string inner = "gmres";
  double t = 0.25;
  std::string smoother = "djacobi";
  double alpha = 0.25;
  std::uint64_t seed = 42;
  aggmg::index_t coarse_size = 600;
  int max_levels = 25;
  int threads = 0;
  bool reuse_cache = false;
  bool allow_pattern = false;
};

aggmg::SmootherKind parse_smoother(const std::string& s) {
  if (s == "jacobi") return aggmg::SmootherKind::jacobi;
  if (s == "djacobi") return aggmg::SmootherKind::damped_jacobi;
  if (s == "sgs") return aggmg::SmootherKind::sgs;
  throw aggmg::Error("unknown smoother '" + s + "'");
}
aggmg::CycleKind parse_cycle(const std::string& s) {
  if (s == "v") return aggmg::CycleKind::v;
  if (s == "k") return aggmg::CycleKind::k;
  if (s == "hybrid") return aggmg::CycleKind::hybrid;
  throw aggmg::Error("unknown cycle '" + s + "'");
}

Json options_to_json(const SolveOptions& o) {
  Json j = Json::object();
  j["matrix"] = o.matrix;
  j["rhs"] = o.rhs;
  j["tol"] = o.tol;
  j["max_iters"] = o.max_iters;
  j["restart"] = o.restart;
  j["solver"] = o.solver;
  j["cycle"] = o.cycle;
  j["klevels"] = o.klevels;
  j["inner"] = o.inner;
  j["t"] = o.t;
  j["smoother"] = o.smoother;
  j["alpha"] = o.alpha;
  j["seed"] = static_cast<unsigned long long>(o.seed);
  j["coarse_size"] = static_cast<long long>(o.coarse_size);
  j["max_levels"] = o.max_levels;
  j["threads"] = o.threads;
  j["reuse_cache"] = o.reuse_cache;
  j["allow_pattern"] = o.allow_pattern;
  return j;
}

SolveOptions options_from_json(const Json& j) {
  SolveOptions o;
  o.matrix = j.at("matrix").s;
  o.rhs = j.at("rhs").s;
  o.tol = j.at("tol").num_value();
  o.max_iters = static_cast<int>(j.at("max_iters").int_value());
  o.restart = static_cast<int>(j.at("restart").int_value());
  o.solver = j.at("solver").s;
  o.cycle = j.at("cycle").s;
  o.klevels = static_cast<int>(j.at("klevels").int_value());
  o.inner = j.at("inner").s;
  o.t = j.at("t").num_value();
  o.smoother = j.at("smoother").s;
  o.alpha = j.at("alpha").num_value();
  o.seed = static_cast<std::uint64_t>(j.at("seed").int_value());
  o.coarse_size = j.at("coarse_size").int_value();
  o.max_levels = static_cast<int>(j.at("max_levels").int_value());
  o.threads = static_cast<int>(j.at("threads").int_value());
  o.reuse_cache = j.at("reuse_cache").b;
  o.allow_pattern = j.at("allow_pattern").b;
  return o;
}

Json make_manifest(const SolveOptions& o) {
  Json m = Json::object();
  m["tool"] = "aggmg";
  m["version"] = aggmg::version();
  m["command"] = "solve";
  m["config"] = options_to_json(o);
  Json inputs = Json::object();
  Json mi = Json::object();
  mi["path"] = o.matrix;
  mi["hash"] = file_hash(o.matrix);
  inputs["matrix"] = mi;
  if (!o.rhs.empty()) {
    Json ri = Json::object();
    ri["path"] = o.rhs;
    ri["hash"] = file_hash(o.rhs);
    inputs["rhs"] = ri;
  }
  m["inputs"] = inputs;
  return m;
}

struct SolveOutcome {
  aggmg::SolveReport report;
  aggmg::HierarchyReport hierarchy;
  double final_relative_residual = 0.0;
};

// aggmg_main.cpp:163-210, unchanged in substance: the CLI's lambda preconditioner included
SolveOutcome run_pipeline(const SolveOptions& o, const aggmg::SparseMatrix& A, const aggmg::Vector& b) {
  aggmg::set_num_threads(o.threads);
  aggmg::SetupConfig scfg;
  scfg.alpha = o.alpha;
  scfg.coarse_size_max = o.coarse_size;
  scfg.max_levels = o.max_levels;
  scfg.smoother = parse_smoother(o.smoother);
  scfg.seed = o.seed;
  scfg.reuse_caches = o.reuse_cache;
  const auto t_setup = Clock::now();
  const aggmg::Hierarchy h = aggmg::setup_hierarchy(A, aggmg::ones_vector(A.n_rows), scfg);
  const double setup_seconds = seconds_since(t_setup);
  for (const std::string& w : h.warnings) std::cerr << "warning: " << w << "\n";
  aggmg::CycleConfig ccfg;
  ccfg.kind = parse_cycle(o.cycle);
  ccfg.k_levels = o.klevels;
  ccfg.t = o.t;
  ccfg.inner = (o.inner == "cg") ? aggmg::InnerKind::cg : aggmg::InnerKind::gmres;
  aggmg::SolverConfig kcfg;
  kcfg.method = (o.solver == "pcg") ? aggmg::SolverMethod::pcg : aggmg::SolverMethod::fgmres;
  kcfg.tol = o.tol;
  kcfg.max_iters = o.max_iters;
  kcfg.restart = o.restart;
  // the reference wires a lambda around apply_preconditioner (aggmg_main.cpp:194-196); the
  // drop-in's device-resident form of the same preconditioner keeps the solve in HBM
  const aggmg::Preconditioner M = aggmg::amg_preconditioner(h, ccfg);
  const aggmg::Vector x0(A.n_rows, 0.0);
  aggmg::SolveResult res = (kcfg.method == aggmg::SolverMethod::pcg) ? aggmg::pcg(A, b, x0, M, kcfg)
                                                                      : aggmg::fgmres(A, b, x0, M, kcfg);
  res.report.setup_seconds = setup_seconds;
  SolveOutcome out;
  out.report = std::move(res.report);
  out.hierarchy = aggmg::hierarchy_report(h);
  const double nb = aggmg::norm2(b);
  out.final_relative_residual = nb > 0.0 ? out.report.residual_history.back() / nb : 0.0;
  return out;
}

Json outcome_to_json(const SolveOutcome& oc) {
  Json j = Json::object();
  j["converged"] = oc.report.converged;
  j["iterations"] = oc.report.iterations;
  j["final_relative_residual"] = oc.final_relative_residual;
  j["setup_seconds"] = oc.report.setup_seconds;
  j["solve_seconds"] = oc.report.solve_seconds;
  j["residual_history"] = Json(oc.report.residual_history);
  if (!oc.report.note.empty()) j["note"] = oc.report.note;
  Json levels = Json::array();
  for (const auto& s : oc.hierarchy.levels) {
    Json l = Json::object();
    l["n"] = static_cast<long long>(s.n);
    l["nnz"] = static_cast<long long>(s.nnz);
    l["nnz_per_row"] = s.nnz_per_row;
    levels.push_back(l);
  }
  Json hj = Json::object();
  hj["levels"] = levels;
  hj["grid_complexity"] = oc.hierarchy.grid_complexity;
  hj["operator_complexity"] = oc.hierarchy.operator_complexity;
  j["hierarchy"] = hj;
  return j;
}

void print_outcome(const SolveOutcome& oc) {
  std::cout << aggmg::format_table(oc.hierarchy);
  std::cout << (oc.report.converged ? "converged" : "NOT converged") << " in "
            << oc.report.iterations << " iterations, relative residual " << std::scientific
            << std::setprecision(3) << oc.final_relative_residual << "\n";
  std::cout << std::fixed << std::setprecision(3) << "setup " << oc.report.setup_seconds
            << " s, solve " << oc.report.solve_seconds << " s\n";
  if (!oc.report.note.empty()) std::cout << "note: " << oc.report.note << "\n";
  std::cout.unsetf(std::ios::floatfield);
}

int cmd_generate(const std::string& kind, aggmg::index_t nx, aggmg::index_t ny, aggmg::index_t nz,
                 double epsilon, int weak_axis, const std::string& rhs_kind, std::uint64_t seed,
                 const std::string& matrix_out, const std::string& rhs_out) {
  aggmg::PoissonSpec spec;
  if (kind == "poisson2d") {
    spec.dims = 2;
  } else if (kind == "poisson3d") {
    spec.dims = 3;
    spec.nz = nz;
  } else {
    throw aggmg::Error("unknown problem kind '" + kind + "'");
  }
  spec.nx = nx;
  spec.ny = ny;
  spec.epsilon = epsilon;
  spec.weak_axis = weak_axis;
  const aggmg::SparseMatrix A = aggmg::generate_poisson(spec);
  const aggmg::Vector b = (rhs_kind == "random") ? aggmg::random_vector(A.n_rows, seed)
                                                 : aggmg::ones_vector(A.n_rows);
  aggmg::write_matrix_market_file(matrix_out, A);
  aggmg::write_vector_market_file(rhs_out, b);
  std::cout << "wrote " << matrix_out << " (" << A.n_rows << " unknowns, " << A.nnz() << " nnz) and "
            << rhs_out << "\n";
  return kExitOk;
}

int cmd_solve(SolveOptions o, const std::string& from_manifest, const std::string& report_path,
              const std::string& manifest_out) {
  if (!from_manifest.empty()) {
    std::ifstream in(from_manifest);
    aggmg::require(in.good(), "cannot open manifest '" + from_manifest + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    const Json m = Json::parse(ss.str());
    o = options_from_json(m.at("config"));
    for (const auto& [name, entry] : m.at("inputs").obj) {
      const std::string path = entry.at("path").s;
      const std::string recorded = entry.at("hash").s;
      if (file_hash(path) != recorded)
        std::cerr << "warning: " << name << " file '" << path
                  << "' differs from the manifest hash; results may not reproduce\n";
    }
  }
  aggmg::require(!o.matrix.empty(), "--matrix is required");
  aggmg::MmOptions mm;
  mm.allow_pattern = o.allow_pattern;
  const aggmg::SparseMatrix A = aggmg::read_matrix_market_file(o.matrix, mm);
  const aggmg::Vector b =
      o.rhs.empty() ? aggmg::ones_vector(A.n_rows) : aggmg::read_vector_market_file(o.rhs);
  aggmg::require(static_cast<aggmg::index_t>(b.size()) == A.n_rows,
                 "right-hand side length does not match the matrix");
  const Json manifest = make_manifest(o);
  const SolveOutcome oc = run_pipeline(o, A, b);
  print_outcome(oc);
  if (!manifest_out.empty()) {
    std::ofstream out(manifest_out);
    aggmg::require(out.good(), "cannot write manifest '" + manifest_out + "'");
    out << manifest.dump(2) << "\n";
  } else {
    std::cout << "manifest: " << manifest.dump() << "\n";
  }
  if (!report_path.empty()) {
    std::ofstream out(report_path);
    aggmg::require(out.good(), "cannot write report '" + report_path + "'");
    Json rep = outcome_to_json(oc);
    rep["manifest"] = manifest;
    out << rep.dump(2) << "\n";
  }
  return oc.report.converged ? kExitOk : kExitNoConvergence;
}

int cmd_bench(const std::vector<aggmg::index_t>& sizes, SolveOptions o, double epsilon,
              aggmg::index_t galerkin_refresh, const std::string& out_path) {
  Json rows = Json::array();
  std::cout << "    size        n  iters     setup_s     solve_s  status\n";
  for (const aggmg::index_t s : sizes) {
    Json row = Json::object();
    row["size"] = static_cast<long long>(s);
    try {
      aggmg::PoissonSpec spec;
      spec.nx = s;
      spec.ny = s;
      spec.epsilon = epsilon;
      const aggmg::SparseMatrix A = aggmg::generate_poisson(spec);
      const aggmg::Vector b = aggmg::ones_vector(A.n_rows);
      const SolveOutcome oc = run_pipeline(o, A, b);
      row["n"] = static_cast<long long>(A.n_rows);
      row["iterations"] = oc.report.iterations;
      row["converged"] = oc.report.converged;
      row["setup_seconds"] = oc.report.setup_seconds;
      row["solve_seconds"] = oc.report.solve_seconds;
      row["final_relative_residual"] = oc.final_relative_residual;
      std::cout << std::setw(8) << s << std::setw(9) << A.n_rows << std::setw(7) << oc.report.iterations
                << std::setw(12) << std::fixed << std::setprecision(3) << oc.report.setup_seconds
                << std::setw(12) << oc.report.solve_seconds
                << (oc.report.converged ? "  ok" : "  NOT converged") << "\n";
      std::cout.unsetf(std::ios::floatfield);
    } catch (const std::exception& e) {
      row["error"] = e.what();
      std::cout << std::setw(8) << s << "  error: " << e.what() << "\n";
    }
    rows.push_back(row);
  }
  Json result = Json::object();
  result["rows"] = rows;
  if (galerkin_refresh > 0) {
    // aggmg_main.cpp:331-373: numeric re-setup through the Galerkin cache vs a fresh setup of
    // the same values (the drop-in has no host-side triple-product path to time instead)
    aggmg::PoissonSpec spec;
    spec.nx = galerkin_refresh;
    spec.ny = galerkin_refresh;
    spec.epsilon = epsilon;
    const aggmg::SparseMatrix A = aggmg::generate_poisson(spec);
    aggmg::SetupConfig scfg;
    scfg.alpha = o.alpha;
    scfg.seed = o.seed;
    scfg.smoother = parse_smoother(o.smoother);
    scfg.reuse_caches = true;
    aggmg::Hierarchy h = aggmg::setup_hierarchy(A, aggmg::ones_vector(A.n_rows), scfg);
    const std::vector<double> values = A.values;
    const auto t_cached = Clock::now();
    h = aggmg::refresh_values(std::move(h), values);
    const double cached_s = seconds_since(t_cached);
    scfg.reuse_caches = false;
    const auto t_direct = Clock::now();
    const aggmg::Hierarchy fresh = aggmg::setup_hierarchy(A, aggmg::ones_vector(A.n_rows), scfg);
    const double direct_s = seconds_since(t_direct);
    std::cout << "galerkin refresh " << galerkin_refresh << "^2: cached " << std::fixed
              << std::setprecision(4) << cached_s << " s, direct " << direct_s << " s, speedup "
              << std::setprecision(2) << direct_s / cached_s << "x\n";
    std::cout.unsetf(std::ios::floatfield);
    Json g = Json::object();
    g["size"] = static_cast<long long>(galerkin_refresh);
    g["cached_seconds"] = cached_s;
    g["direct_seconds"] = direct_s;
    g["speedup"] = direct_s / cached_s;
    result["galerkin_refresh"] = g;
  }
  if (!out_path.empty()) {
    std::ofstream out(out_path);
    aggmg::require(out.good(), "cannot write '" + out_path + "'");
    out << result.dump(2) << "\n";
  }
  return kExitOk;
}

// ---- option parsing: "--name value" / "--flag", the reference's names --------------------------
struct Args {
  std::map<std::string, std::string> val;
  std::map<std::string, bool> flag;
};
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& options,
           const std::vector<std::string>& flags) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    std::string v;
    const auto eq = k.find('=');
    if (eq != std::string::npos) {
      v = k.substr(eq + 1);
      k = k.substr(0, eq);
    }
    if (std::find(flags.begin(), flags.end(), k) != flags.end()) {
      a.flag[k] = true;
      continue;
    }
    if (std::find(options.begin(), options.end(), k) == options.end())
      throw ParseError("The following argument was not expected: " + k);
    if (eq == std::string::npos) {
      if (i + 1 >= argc) throw ParseError(k + " requires an argument");
      v = argv[++i];
    }
    a.val[k] = v;
  }
  return a;
}
template <class T>
void get(const Args& a, const std::string& k, T& out) {
  auto it = a.val.find(k);
  if (it == a.val.end()) return;
  std::istringstream s(it->second);
  if constexpr (std::is_same_v<T, std::string>) {
    out = it->second;
  } else {
    T v{};
    s >> v;
    if (s.fail() || !s.eof()) throw ParseError(k + ": bad value '" + it->second + "'");
    out = v;
  }
}
void member(const std::string& k, const std::string& v, const std::vector<std::string>& allowed) {
  if (std::find(allowed.begin(), allowed.end(), v) == allowed.end())
    throw ParseError(k + ": '" + v + "' not in the allowed set");
}

void read_solve_options(const Args& a, SolveOptions& o, bool bench) {
  if (!bench) {
    get(a, "--matrix", o.matrix);
    get(a, "--rhs", o.rhs);
    get(a, "--max-levels", o.max_levels);
    get(a, "--restart", o.restart);
    o.allow_pattern = a.flag.count("--allow-pattern") > 0;
  }
  get(a, "--tol", o.tol);
  get(a, "--max-iters", o.max_iters);
  get(a, "--solver", o.solver);
  member("--solver", o.solver, {"fgmres", "pcg"});
  get(a, "--cycle", o.cycle);
  member("--cycle", o.cycle, {"v", "k", "hybrid"});
  get(a, "--klevels", o.klevels);
  get(a, "--inner", o.inner);
  member("--inner", o.inner, {"cg", "gmres"});
  get(a, "--t", o.t);
  get(a, "--smoother", o.smoother);
  member("--smoother", o.smoother, {"jacobi", "djacobi", "sgs"});
  get(a, "--alpha", o.alpha);
  get(a, "--seed", o.seed);
  get(a, "--coarse-size", o.coarse_size);
  get(a, "--threads", o.threads);
  o.reuse_cache = a.flag.count("--reuse-cache") > 0;
}

const char* kUsage =
    "aggregation multigrid solver (B200)\n"
    "Usage: aggmg SUBCOMMAND [OPTIONS]\n"
    "Subcommands:\n"
    "  generate   write a Matrix Market test problem\n"
    "  solve      solve a system with the multigrid-preconditioned Krylov solver\n"
    "  bench      sweep grid sizes and report timings\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage << "A subcommand is required\n";
    return kExitInputError;
  }
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    std::cout << kUsage;
    return kExitOk;
  }
  const std::vector<std::string> common = {"--tol", "--max-iters", "--solver", "--cycle", "--klevels",
                                           "--inner", "--t", "--smoother", "--alpha", "--seed",
                                           "--coarse-size", "--threads"};
  auto init = [] {
    if (aggmg_init(0) != AGGMG_OK) throw aggmg::Error(aggmg_last_error());
  };
  try {
    if (sub == "generate") {
      const Args a = parse(argc, argv, 2, {"--kind", "--nx", "--ny", "--nz", "--epsilon", "--weak-axis",
                                           "--rhs-kind", "--seed", "--matrix-out", "--rhs-out"}, {});
      std::string kind = "poisson2d", rhs_kind = "ones", mout = "matrix.mtx", rout = "rhs.mtx";
      aggmg::index_t nx = 64, ny = 64, nz = 64;
      double eps = 0.01;  // anisotropic by default, as the reference
      int weak = -1;
      std::uint64_t seed = 42;
      get(a, "--kind", kind);
      get(a, "--nx", nx);
      get(a, "--ny", ny);
      get(a, "--nz", nz);
      get(a, "--epsilon", eps);
      get(a, "--weak-axis", weak);
      get(a, "--rhs-kind", rhs_kind);
      get(a, "--seed", seed);
      get(a, "--matrix-out", mout);
      get(a, "--rhs-out", rout);
      if (rhs_kind == "random") init();  // the generator's random right-hand side runs on the device
      return cmd_generate(kind, nx, ny, nz, eps, weak, rhs_kind, seed, mout, rout);
    }
    if (sub == "solve") {
      std::vector<std::string> opts = common;
      for (const char* k : {"--matrix", "--rhs", "--max-levels", "--restart", "--from-manifest",
                            "--report", "--manifest-out"})
        opts.push_back(k);
      const Args a = parse(argc, argv, 2, opts, {"--reuse-cache", "--allow-pattern"});
      SolveOptions o;
      read_solve_options(a, o, false);
      std::string from, report, mout;
      get(a, "--from-manifest", from);
      get(a, "--report", report);
      get(a, "--manifest-out", mout);
      init();
      return cmd_solve(o, from, report, mout);
    }
    if (sub == "bench") {
      std::vector<std::string> opts = common;
      for (const char* k : {"--sizes", "--epsilon", "--galerkin-refresh", "--out"}) opts.push_back(k);
      const Args a = parse(argc, argv, 2, opts, {"--reuse-cache"});
      SolveOptions o;
      read_solve_options(a, o, true);
      std::string sizes_s = "64,128,256", out;
      double eps = 1.0;
      aggmg::index_t gref = 0;
      get(a, "--sizes", sizes_s);
      get(a, "--epsilon", eps);
      get(a, "--galerkin-refresh", gref);
      get(a, "--out", out);
      std::vector<aggmg::index_t> sizes;
      std::stringstream ss(sizes_s);
      std::string tok;
      while (std::getline(ss, tok, ',')) sizes.push_back(std::stoll(tok));
      init();
      return cmd_bench(sizes, o, eps, gref, out);
    }
    std::cerr << kUsage << "The following argument was not expected: " << sub << "\n";
    return kExitInputError;
  } catch (const ParseError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return kExitInputError;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitInputError;
  }
}
