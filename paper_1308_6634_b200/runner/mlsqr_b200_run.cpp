// mlsqr_b200_run.cpp -- the reference's experiment harness (`mlsqr run | compare`,
// tools/main.cpp:1-74) on the B200 path: the same configuration schema (config.cpp:1-309,
// config.hpp:1-71), the same artifacts (runner.cpp:55-121, 301-325: trace.csv, solution.csv,
// basis_###.csv, solution_outer_###.csv, meta.json) and the same exit codes, with every
// operator, SpdMap and Krylov solve running on the device through the C-ABI
// (include/mlsqr_b200.h).  Host work is input generation (problems.cpp conventions),
// bookkeeping and formatting, as in the reference's runner.
//
// B200 extension of the schema: solver.spd.mode = "vcycle" (the multigrid SpdMap, with the
// optional keys levels / nu_pre / nu_post / coarse_sweeps / omega).  "cholesky" and
// "inner_cg" are the reference's SpdSolver modes, run on the device.
#include <json.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/mlsqr_b200.h"

namespace fs = std::filesystem;
using nlohmann::json;

namespace {

// ---------------------------------------------------------------------------
// errors (errors.hpp:9-41 + ConfigError) and C-ABI status mapping
// ---------------------------------------------------------------------------
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SolverFailure : std::runtime_error {  // BreakdownError / FactorizationError
  using std::runtime_error::runtime_error;
};

void check(int st) {
  if (st == MLSQR_OK) return;
  const std::string msg = mlsqr_last_error();
  if (st == MLSQR_EBREAKDOWN || st == MLSQR_EFACTOR) throw SolverFailure(msg);
  if (st == MLSQR_EINVAL || st == MLSQR_EDIM) throw std::invalid_argument(msg);
  throw std::runtime_error("mlsqr_b200 status " + std::to_string(st) + ": " + msg);
}

// ---------------------------------------------------------------------------
// configuration (config.hpp:16-67), parsed exactly like config.cpp
// ---------------------------------------------------------------------------
struct Shape2D {
  bool disk = false;
  double x0 = 0, y0 = 0, x1 = 0, y1 = 0, cx = 0, cy = 0, r = 0, value = 1.0;
};

struct ProblemConfig {
  bool deblur2d = false;
  size_t n = 512, nx = 64, ny = 64;
  double sigma_f = 0.03, sigma_n = 0.01;
  uint64_t seed = 0;
  std::optional<std::vector<std::pair<double, double>>> phantom1d;
  std::optional<std::vector<Shape2D>> phantom2d;
  json raw;
};

enum class Method { lsqr, mlsqr, cg_normal, lagged_diffusivity };
enum class SpdMode { cholesky, inner_cg, vcycle };

struct SolverConfig {
  Method method = Method::lsqr;
  double tau = 0.0;
  int pen_kind = MLSQR_PEN_TIKHONOV;
  double T = 1.0;
  bool penalty_given = false;
  std::string regularizer = "ideal";
  mlsqr_stop stopping{};
  SpdMode spd_mode = SpdMode::cholesky;
  int k_inner = 30;
  int mg_levels = 3, nu_pre = 2, nu_post = 2, coarse_sweeps = 4;
  double omega = 2.0 / 3.0;
  std::optional<double> epsilon;
  int inner_cap = 20;
  double rel_decrease_threshold = 0.15;
  int max_outer = 25;
  bool store_basis = false;
};

struct OutputConfig {
  std::string directory = "out";
  bool traces = true, solutions = true, outer_snapshots = false;
  int basis_vectors = 0;
};

struct ExperimentConfig {
  ProblemConfig problem;
  SolverConfig solver;
  OutputConfig output;
};

void reject_unknown(const json& obj, const char* section, std::initializer_list<const char*> allowed) {
  for (auto it = obj.begin(); it != obj.end(); ++it) {
    if (std::find_if(allowed.begin(), allowed.end(), [&](const char* k) { return it.key() == k; }) ==
        allowed.end())
      throw ConfigError("unknown key '" + it.key() + "' in " + section);
  }
}

const json& need(const json& obj, const char* section, const char* key) {
  const auto it = obj.find(key);
  if (it == obj.end()) throw ConfigError(std::string("missing key '") + key + "' in " + section);
  return *it;
}

double as_number(const json& v, const char* key) {
  if (!v.is_number()) throw ConfigError(std::string("key '") + key + "' must be a number");
  return v.get<double>();
}

size_t as_count(const json& v, const char* key) {
  if (!v.is_number_integer() || v.get<long long>() < 0)
    throw ConfigError(std::string("key '") + key + "' must be a nonnegative integer");
  return v.get<size_t>();
}

int as_positive_int(const json& v, const char* key) {
  if (!v.is_number_integer() || v.get<long long>() < 1)
    throw ConfigError(std::string("key '") + key + "' must be a positive integer");
  return v.get<int>();
}

bool as_bool(const json& v, const char* key) {
  if (!v.is_boolean()) throw ConfigError(std::string("key '") + key + "' must be a boolean");
  return v.get<bool>();
}

std::string as_string(const json& v, const char* key) {
  if (!v.is_string()) throw ConfigError(std::string("key '") + key + "' must be a string");
  return v.get<std::string>();
}

// Phantom1D::validate (problems.cpp:46-63)
void validate_phantom1d(const std::vector<std::pair<double, double>>& jumps) {
  if (jumps.empty()) throw std::invalid_argument("phantom needs at least one plateau");
  double last = -1.0;
  for (const auto& [pos, level] : jumps) {
    (void)level;
    if (!(pos >= 0.0 && pos <= 1.0)) throw std::invalid_argument("phantom positions must lie in [0, 1]");
    if (!(pos > last)) throw std::invalid_argument("phantom positions must be strictly increasing");
    last = pos;
  }
  if (jumps.front().first != 0.0) throw std::invalid_argument("phantom must define the level at position 0");
}

// Phantom2D::validate (problems.cpp:102-113)
void validate_phantom2d(const std::vector<Shape2D>& shapes) {
  for (const Shape2D& s : shapes) {
    if (!s.disk) {
      if (!(s.x1 > s.x0 && s.y1 > s.y0)) throw std::invalid_argument("degenerate rectangle in phantom");
    } else if (!(s.r > 0.0)) {
      throw std::invalid_argument("disk radius must be positive");
    }
  }
}

std::vector<std::pair<double, double>> parse_phantom1d(const json& arr) {  // config.cpp:60-79
  if (!arr.is_array()) throw ConfigError("key 'phantom' must be an array of [position, level]");
  std::vector<std::pair<double, double>> p;
  for (const json& item : arr) {
    if (!item.is_array() || item.size() != 2)
      throw ConfigError("each 'phantom' entry must be a [position, level] pair");
    p.emplace_back(as_number(item[0], "phantom position"), as_number(item[1], "phantom level"));
  }
  try {
    validate_phantom1d(p);
  } catch (const std::invalid_argument& e) {
    throw ConfigError(std::string("invalid 'phantom': ") + e.what());
  }
  return p;
}

std::vector<Shape2D> parse_phantom2d(const json& arr) {  // config.cpp:81-113
  if (!arr.is_array()) throw ConfigError("key 'phantom' must be an array of shapes");
  std::vector<Shape2D> p;
  for (const json& item : arr) {
    if (!item.is_object()) throw ConfigError("each 'phantom' entry must be a shape object");
    Shape2D s;
    const std::string kind = as_string(need(item, "phantom shape", "shape"), "shape");
    if (kind == "rect") {
      reject_unknown(item, "phantom shape", {"shape", "x0", "y0", "x1", "y1", "value"});
      s.x0 = as_number(need(item, "phantom shape", "x0"), "x0");
      s.y0 = as_number(need(item, "phantom shape", "y0"), "y0");
      s.x1 = as_number(need(item, "phantom shape", "x1"), "x1");
      s.y1 = as_number(need(item, "phantom shape", "y1"), "y1");
    } else if (kind == "disk") {
      reject_unknown(item, "phantom shape", {"shape", "cx", "cy", "r", "value"});
      s.disk = true;
      s.cx = as_number(need(item, "phantom shape", "cx"), "cx");
      s.cy = as_number(need(item, "phantom shape", "cy"), "cy");
      s.r = as_number(need(item, "phantom shape", "r"), "r");
    } else {
      throw ConfigError("key 'shape' must be 'rect' or 'disk'");
    }
    s.value = as_number(need(item, "phantom shape", "value"), "value");
    p.push_back(s);
  }
  try {
    validate_phantom2d(p);
  } catch (const std::invalid_argument& e) {
    throw ConfigError(std::string("invalid 'phantom': ") + e.what());
  }
  return p;
}

ProblemConfig parse_problem(const json& obj) {  // config.cpp:115-141
  if (!obj.is_object()) throw ConfigError("'problem' must be an object");
  ProblemConfig p;
  p.raw = obj;
  const std::string type = as_string(need(obj, "problem", "type"), "type");
  if (type == "deconv1d") {
    reject_unknown(obj, "problem", {"type", "n", "sigma_f", "sigma_n", "seed", "phantom"});
    p.n = as_count(need(obj, "problem", "n"), "n");
    if (p.n < 2) throw ConfigError("key 'n' must be at least 2");
    if (obj.contains("phantom")) p.phantom1d = parse_phantom1d(obj["phantom"]);
  } else if (type == "deblur2d") {
    reject_unknown(obj, "problem", {"type", "nx", "ny", "sigma_f", "sigma_n", "seed", "phantom"});
    p.deblur2d = true;
    p.nx = as_count(need(obj, "problem", "nx"), "nx");
    p.ny = as_count(need(obj, "problem", "ny"), "ny");
    if (p.nx < 2 || p.ny < 2) throw ConfigError("keys 'nx'/'ny' must be at least 2");
    if (obj.contains("phantom")) p.phantom2d = parse_phantom2d(obj["phantom"]);
  } else {
    throw ConfigError("key 'type' must be 'deconv1d' or 'deblur2d'");
  }
  p.sigma_f = as_number(need(obj, "problem", "sigma_f"), "sigma_f");
  if (!(p.sigma_f > 0.0)) throw ConfigError("key 'sigma_f' must be positive");
  p.sigma_n = as_number(need(obj, "problem", "sigma_n"), "sigma_n");
  if (!(p.sigma_n >= 0.0)) throw ConfigError("key 'sigma_n' must be nonnegative");
  p.seed = as_count(need(obj, "problem", "seed"), "seed");
  return p;
}

int parse_penalty_kind(const std::string& kind) {  // config.cpp:143-149
  if (kind == "tikhonov") return MLSQR_PEN_TIKHONOV;
  if (kind == "tv_smoothed") return MLSQR_PEN_TV;
  if (kind == "pm_log") return MLSQR_PEN_PM_LOG;
  if (kind == "pm_exp") return MLSQR_PEN_PM_EXP;
  throw ConfigError("key 'kind' must be one of tikhonov, tv_smoothed, pm_log, pm_exp");
}

// StoppingConfig::validate (krylov.cpp:219-226)
void validate_stop(const mlsqr_stop& s) {
  if (s.max_iters < 1) throw std::invalid_argument("max_iters must be at least 1");
  if (s.use_s4 && !(s.eta > 1.0)) throw std::invalid_argument("discrepancy stopping needs a safety factor eta > 1");
  if (s.use_s4 && !(s.delta >= 0.0)) throw std::invalid_argument("noise level delta must be >= 0");
  if (!(s.atol >= 0.0 && s.btol >= 0.0)) throw std::invalid_argument("tolerances must be >= 0");
}

mlsqr_stop parse_stopping(const json& obj) {  // config.cpp:151-178
  if (!obj.is_object()) throw ConfigError("'stopping' must be an object");
  reject_unknown(obj, "stopping", {"criteria", "atol", "btol", "conlim", "delta", "eta", "max_iters"});
  mlsqr_stop s{};  // StoppingConfig defaults (krylov.hpp:19-36)
  s.atol = 1e-8;
  s.btol = 1e-8;
  s.conlim = 1e8;
  s.delta = 0.0;
  s.eta = 1.1;
  s.max_iters = 100;
  const json& crit = need(obj, "stopping", "criteria");
  if (!crit.is_array()) throw ConfigError("key 'criteria' must be an array");
  for (const json& c : crit) {
    const std::string name = as_string(c, "criteria");
    if (name == "S1") s.use_s1 = 1;
    else if (name == "S2") s.use_s2 = 1;
    else if (name == "S3") s.use_s3 = 1;
    else if (name == "S4") s.use_s4 = 1;
    else throw ConfigError("key 'criteria' allows S1, S2, S3, S4 (iteration cap is implicit)");
  }
  if (obj.contains("atol")) s.atol = as_number(obj["atol"], "atol");
  if (obj.contains("btol")) s.btol = as_number(obj["btol"], "btol");
  if (obj.contains("conlim")) s.conlim = as_number(obj["conlim"], "conlim");
  if (obj.contains("delta")) s.delta = as_number(obj["delta"], "delta");
  if (obj.contains("eta")) s.eta = as_number(obj["eta"], "eta");
  s.max_iters = as_positive_int(need(obj, "stopping", "max_iters"), "max_iters");
  try {
    validate_stop(s);
  } catch (const std::invalid_argument& e) {
    throw ConfigError(std::string("invalid 'stopping': ") + e.what());
  }
  return s;
}

SolverConfig parse_solver(const json& obj) {  // config.cpp:180-259
  if (!obj.is_object()) throw ConfigError("'solver' must be an object");
  reject_unknown(obj, "solver",
                 {"method", "tau", "penalty", "regularizer", "stopping", "spd", "epsilon", "inner_cap",
                  "rel_decrease_threshold", "max_outer", "store_basis"});
  SolverConfig s;
  const std::string method = as_string(need(obj, "solver", "method"), "method");
  if (method == "lsqr") s.method = Method::lsqr;
  else if (method == "mlsqr") s.method = Method::mlsqr;
  else if (method == "cg_normal") s.method = Method::cg_normal;
  else if (method == "lagged_diffusivity") s.method = Method::lagged_diffusivity;
  else throw ConfigError("key 'method' must be lsqr, mlsqr, cg_normal or lagged_diffusivity");
  if (obj.contains("tau")) {
    s.tau = as_number(obj["tau"], "tau");
    if (!(s.tau >= 0.0)) throw ConfigError("key 'tau' must be nonnegative");
  }
  if (obj.contains("penalty")) {
    const json& pen = obj["penalty"];
    if (!pen.is_object()) throw ConfigError("'penalty' must be an object");
    reject_unknown(pen, "penalty", {"kind", "T"});
    const int kind = parse_penalty_kind(as_string(need(pen, "penalty", "kind"), "kind"));
    double threshold = 1.0;
    if (kind != MLSQR_PEN_TIKHONOV) {
      threshold = as_number(need(pen, "penalty", "T"), "T");
      if (!(threshold > 0.0)) throw ConfigError("key 'T' must be positive");
    } else if (pen.contains("T")) {
      threshold = as_number(pen["T"], "T");
    }
    s.pen_kind = kind;
    s.T = threshold;
    s.penalty_given = true;
  }
  if (obj.contains("regularizer")) {
    s.regularizer = as_string(obj["regularizer"], "regularizer");
    if (s.regularizer != "ideal" && s.regularizer != "laplacian")
      throw ConfigError("key 'regularizer' must be 'ideal' or 'laplacian'");
  }
  s.stopping = parse_stopping(need(obj, "solver", "stopping"));
  if (obj.contains("spd")) {
    const json& spd = obj["spd"];
    if (!spd.is_object()) throw ConfigError("'spd' must be an object");
    const std::string mode = as_string(need(spd, "spd", "mode"), "mode");
    if (mode == "cholesky") s.spd_mode = SpdMode::cholesky;
    else if (mode == "inner_cg") s.spd_mode = SpdMode::inner_cg;
    else if (mode == "vcycle") s.spd_mode = SpdMode::vcycle;  // B200 extension
    else throw ConfigError("key 'mode' must be 'cholesky', 'inner_cg' or 'vcycle'");
    if (s.spd_mode == SpdMode::vcycle) {
      reject_unknown(spd, "spd", {"mode", "levels", "nu_pre", "nu_post", "coarse_sweeps", "omega"});
      if (spd.contains("levels")) s.mg_levels = as_positive_int(spd["levels"], "levels");
      if (spd.contains("nu_pre")) s.nu_pre = as_positive_int(spd["nu_pre"], "nu_pre");
      if (spd.contains("nu_post")) s.nu_post = as_positive_int(spd["nu_post"], "nu_post");
      // M^-1 must be a symmetric map (spdsolve.hpp:11-14): the post-smoother mirrors the pre-smoother
      if (s.nu_post != s.nu_pre) throw ConfigError("keys 'nu_pre' and 'nu_post' must be equal (a symmetric V-cycle)");
      if (spd.contains("coarse_sweeps")) s.coarse_sweeps = as_positive_int(spd["coarse_sweeps"], "coarse_sweeps");
      if (spd.contains("omega")) {
        s.omega = as_number(spd["omega"], "omega");
        if (!(s.omega > 0.0)) throw ConfigError("key 'omega' must be positive");
      }
    } else {
      reject_unknown(spd, "spd", {"mode", "k_inner"});
      if (spd.contains("k_inner")) s.k_inner = as_positive_int(spd["k_inner"], "k_inner");
    }
  }
  if (obj.contains("epsilon")) {
    const json& eps = obj["epsilon"];
    if (eps.is_string()) {
      if (eps.get<std::string>() != "auto") throw ConfigError("key 'epsilon' must be a number or 'auto'");
    } else {
      const double value = as_number(eps, "epsilon");
      if (!(value >= 0.0)) throw ConfigError("key 'epsilon' must be nonnegative");
      s.epsilon = value;
    }
  }
  if (obj.contains("inner_cap")) s.inner_cap = as_positive_int(obj["inner_cap"], "inner_cap");
  if (obj.contains("rel_decrease_threshold")) {
    s.rel_decrease_threshold = as_number(obj["rel_decrease_threshold"], "rel_decrease_threshold");
    if (!(s.rel_decrease_threshold > 0.0 && s.rel_decrease_threshold < 1.0))
      throw ConfigError("key 'rel_decrease_threshold' must lie in (0, 1)");
  }
  if (obj.contains("max_outer")) s.max_outer = as_positive_int(obj["max_outer"], "max_outer");
  if (obj.contains("store_basis")) s.store_basis = as_bool(obj["store_basis"], "store_basis");
  if (s.method != Method::lsqr && !s.penalty_given)
    throw ConfigError(std::string("method '") + method + "' requires a 'penalty' section");
  return s;
}

OutputConfig parse_output(const json& obj) {  // config.cpp:261-278
  if (!obj.is_object()) throw ConfigError("'output' must be an object");
  reject_unknown(obj, "output", {"directory", "traces", "solutions", "basis_vectors", "outer_snapshots"});
  OutputConfig o;
  o.directory = as_string(need(obj, "output", "directory"), "directory");
  if (obj.contains("traces")) o.traces = as_bool(obj["traces"], "traces");
  if (obj.contains("solutions")) o.solutions = as_bool(obj["solutions"], "solutions");
  if (obj.contains("basis_vectors")) o.basis_vectors = static_cast<int>(as_count(obj["basis_vectors"], "basis_vectors"));
  if (obj.contains("outer_snapshots")) o.outer_snapshots = as_bool(obj["outer_snapshots"], "outer_snapshots");
  return o;
}

ExperimentConfig parse_config(const json& doc) {  // config.cpp:282-291
  if (!doc.is_object()) throw ConfigError("configuration root must be an object");
  reject_unknown(doc, "configuration root", {"problem", "solver", "output"});
  ExperimentConfig cfg;
  cfg.problem = parse_problem(need(doc, "configuration root", "problem"));
  cfg.solver = parse_solver(need(doc, "configuration root", "solver"));
  cfg.output = parse_output(need(doc, "configuration root", "output"));
  return cfg;
}

ExperimentConfig load_config(const fs::path& path) {  // config.cpp:293-303
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open config file: " + path.string());
  json doc;
  try {
    in >> doc;
  } catch (const json::parse_error& e) {
    throw ConfigError("config is not valid JSON: " + std::string(e.what()));
  }
  return parse_config(doc);
}

const char* method_name(Method m) {
  switch (m) {
    case Method::lsqr: return "lsqr";
    case Method::mlsqr: return "mlsqr";
    case Method::cg_normal: return "cg_normal";
    case Method::lagged_diffusivity: return "lagged_diffusivity";
  }
  return "unknown";
}

const char* stop_name(int r) {  // to_string(StopReason)
  static const char* names[] = {"S1", "S2", "S3", "S4", "max_iters", "breakdown"};
  return r >= 0 && r <= 5 ? names[r] : "unknown";
}

// ---------------------------------------------------------------------------
// device objects (RAII over the C-ABI)
// ---------------------------------------------------------------------------
struct Ctx {
  mlsqr_ctx* h = nullptr;
  Ctx() { check(mlsqr_ctx_create(0, nullptr, &h)); }
  ~Ctx() { mlsqr_ctx_destroy(h); }
};
struct Op {
  mlsqr_op* h = nullptr;
  ~Op() { mlsqr_op_destroy(h); }
};
struct Pc {
  mlsqr_pc* h = nullptr;
  Pc() = default;
  Pc(const Pc&) = delete;
  Pc& operator=(const Pc&) = delete;
  ~Pc() { mlsqr_pc_destroy(h); }
};

// ---------------------------------------------------------------------------
// the experiment bundle (problems.hpp:52-85, runner.cpp:28-36)
// ---------------------------------------------------------------------------
struct Bundle {
  int dims = 1;
  size_t nx = 0, ny = 1, n = 0;
  double h = 0.0;                 // Grid::spacing
  double data_cell_measure = 1.0;
  std::vector<double> f_true, g;
  Op op;
};

std::vector<double> taps_for(size_t n, double sigma_f) {
  int r = 0;
  check(mlsqr_taps(n, sigma_f, 1.0, -1, nullptr, &r));  // R = ceil(6 sigma / h) (linop.cpp:96)
  std::vector<double> t(2 * (size_t)r + 1);
  check(mlsqr_taps(n, sigma_f, 1.0, r, t.data(), &r));
  return t;
}

// Phantom1D::default_phantom (problems.cpp:31-44) / realize (:65-79)
std::vector<double> realize1d(const std::vector<std::pair<double, double>>& jumps, size_t n) {
  std::vector<double> f(n);
  const double h = 1.0 / static_cast<double>(n);
  for (size_t i = 0; i < n; ++i) {
    const double x = (static_cast<double>(i) + 0.5) * h;
    double level = jumps.front().second;
    for (const auto& [pos, lev] : jumps)
      if (pos <= x) level = lev;
    f[i] = level;
  }
  return f;
}

std::vector<std::pair<double, double>> default_phantom1d() {
  return {{0.00, 0.0}, {0.10, 1.0}, {0.28, 0.0}, {0.40, 1.5}, {0.62, 0.2}, {0.76, 2.0}, {0.80, 0.2}, {0.90, 0.0}};
}

// Phantom2D::default_phantom (problems.cpp:81-100) / realize (:115-133)
std::vector<Shape2D> default_phantom2d() {
  Shape2D d1, d2, r1;
  d1.disk = true, d1.cx = 0.30, d1.cy = 0.35, d1.r = 0.13, d1.value = 1.0;
  d2.disk = true, d2.cx = 0.70, d2.cy = 0.65, d2.r = 0.10, d2.value = 1.0;
  r1.x0 = 0.55, r1.y0 = 0.15, r1.x1 = 0.85, r1.y1 = 0.35, r1.value = 0.6;
  return {d1, d2, r1};
}

std::vector<double> realize2d(const std::vector<Shape2D>& shapes, size_t nx, size_t ny) {
  std::vector<double> f(nx * ny, 0.0);
  const double hx = 1.0 / static_cast<double>(nx), hy = 1.0 / static_cast<double>(ny);
  for (size_t iy = 0; iy < ny; ++iy) {
    const double y = (static_cast<double>(iy) + 0.5) * hy;
    for (size_t ix = 0; ix < nx; ++ix) {
      const double x = (static_cast<double>(ix) + 0.5) * hx;
      for (const Shape2D& s : shapes) {
        const bool inside = !s.disk ? (x >= s.x0 && x <= s.x1 && y >= s.y0 && y <= s.y1)
                                    : ((x - s.cx) * (x - s.cx) + (y - s.cy) * (y - s.cy) <= s.r * s.r);
        if (inside) f[iy * nx + ix] = s.value;
      }
    }
  }
  return f;
}

// make_deconv1d / make_deblur2d (problems.cpp:135-185): g = A f_true (+ seeded noise)
void build_bundle(Ctx& ctx, const ProblemConfig& p, uint64_t seed, Bundle& b) {
  if (!p.deblur2d) {
    b.dims = 1;
    b.nx = b.n = p.n;
    b.h = 1.0 / static_cast<double>(p.n);
    b.data_cell_measure = b.h;
    const std::vector<double> t = taps_for(p.n, p.sigma_f);
    check(mlsqr_blur_create(ctx.h, 1, p.n, 1, 1, t.data(), static_cast<int>(t.size() / 2), &b.op.h));
    b.f_true = realize1d(p.phantom1d.value_or(default_phantom1d()), p.n);
  } else {
    b.dims = 2;
    b.nx = p.nx;
    b.ny = p.ny;
    b.n = p.nx * p.ny;
    b.h = 1.0 / static_cast<double>(p.nx);  // Grid::plane(nx, ny, hx)
    b.data_cell_measure = b.h * (1.0 / static_cast<double>(p.ny));
    const std::vector<double> tx = taps_for(p.nx, p.sigma_f), ty = taps_for(p.ny, p.sigma_f);
    if (p.nx == p.ny)
      check(mlsqr_blur_create(ctx.h, 2, p.nx, p.ny, 1, tx.data(), static_cast<int>(tx.size() / 2), &b.op.h));
    else
      check(mlsqr_blur2d_create_axes(ctx.h, p.nx, p.ny, tx.data(), static_cast<int>(tx.size() / 2), ty.data(),
                                     static_cast<int>(ty.size() / 2), &b.op.h));
    b.f_true = realize2d(p.phantom2d.value_or(default_phantom2d()), p.nx, p.ny);
  }
  b.g.assign(b.n, 0.0);
  check(mlsqr_op_apply(b.op.h, b.f_true.data(), b.n, b.g.data(), b.n, MLSQR_HOST));
  if (p.sigma_n > 0.0) {
    std::vector<double> nv(b.n);
    check(mlsqr_gauss_fill(seed, b.n, p.sigma_n, nv.data()));
    for (size_t i = 0; i < b.n; ++i) b.g[i] += 1.0 * nv[i];  // kernels::axpy(1.0, n, g)
  }
}

// M holder: a V-cycle map (levels = 1 unless the vcycle SpdMap is wanted) whose level 0 is
// assemble_m(grid, field, penalty) + eps I (diffusion.cpp:59-87); returns eps used
double assemble_m(Ctx& ctx, const Bundle& b, const SolverConfig& s, const std::vector<double>& field,
                  std::optional<double> eps, int levels, Pc& m) {
  check(mlsqr_vcycle_create(ctx.h, b.dims, b.nx, b.ny, 1, b.h, levels, s.nu_pre, s.nu_post, s.omega,
                            s.coarse_sweeps, &m.h));
  double used = 0.0;
  check(mlsqr_vcycle_update(m.h, field.data(), MLSQR_HOST, s.pen_kind, s.T, eps ? *eps : -1.0, &used));
  return used;
}

// the SpdMap of a mode over an M holder (SpdSolver::factorize / inner_cg, or the V-cycle)
mlsqr_pc* spd_solver(const SolverConfig& s, Pc& m, Pc& owned) {
  if (s.spd_mode == SpdMode::vcycle) return m.h;
  if (s.spd_mode == SpdMode::cholesky) check(mlsqr_chol_map_create(m.h, &owned.h, nullptr));
  else check(mlsqr_inner_cg_map_create(m.h, s.k_inner, &owned.h));
  return owned.h;
}

std::string fmt(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

double error_norm(const std::vector<double>& f, const std::vector<double>& t) {  // problems.cpp:187-198
  double acc = 0.0;
  for (size_t i = 0; i < f.size(); ++i) {
    const double d = f[i] - t[i];
    acc += d * d;
  }
  return std::sqrt(acc);
}

double penalty_R(Ctx& ctx, const Bundle& b, const SolverConfig& s, const double* f) {
  double v = 0.0;  // penalty_functional (diffusion.cpp:89-101) on the device
  check(mlsqr_penalty_functional(ctx.h, b.dims, b.nx, b.ny, 1, b.h, f, MLSQR_HOST, s.pen_kind, s.T, &v));
  return v;
}

// one solve's results (SolveResult, krylov.hpp:69-75)
struct Solve {
  std::vector<double> f;
  std::vector<mlsqr_iter_rec> trace;
  std::vector<double> snaps;  // iterations x n
  mlsqr_solve_info info{};
};

Solve run_krylov(const Bundle& b, mlsqr_pc* pc, double tau, const mlsqr_stop& stop, bool snapshots,
                 bool cgn) {
  Solve r;
  r.f.assign(b.n, 0.0);
  r.trace.resize((size_t)stop.max_iters);
  if (snapshots) r.snaps.resize((size_t)stop.max_iters * b.n);
  std::vector<double> al((size_t)stop.max_iters + 1), be((size_t)stop.max_iters + 2);
  mlsqr_solve_opts o{};
  o.record_snapshots = snapshots ? 1 : 0;
  o.snapshots = snapshots ? r.snaps.data() : nullptr;
  if (cgn)
    check(mlsqr_cg_normal_solve_with(b.op.h, pc, b.g.data(), tau, &stop, &o, r.f.data(), r.trace.data(), &r.info,
                                     MLSQR_HOST));
  else
    check(mlsqr_solve_with(b.op.h, pc, b.g.data(), tau, &stop, &o, r.f.data(), r.trace.data(), al.data(),
                           be.data(), &r.info, MLSQR_HOST));
  r.trace.resize((size_t)r.info.iterations);
  if (snapshots) r.snaps.resize((size_t)r.info.iterations * b.n);
  return r;
}

struct TraceRow {
  int outer_k, inner_i;
  mlsqr_iter_rec rec;
  const double* snapshot;  // may be null
};

void write_trace(Ctx& ctx, const fs::path& path, const std::vector<TraceRow>& rows, const Bundle& b,
                 const SolverConfig& s) {  // runner.cpp:55-73
  std::ofstream out(path);
  out << "outer_k,inner_i,res_data,res_damped,s2_estimate,anorm_est,cond_est,penalty_R,"
         "error_norm_if_truth_known\n";
  for (const TraceRow& row : rows) {
    double pv = std::numeric_limits<double>::quiet_NaN(), err = pv;
    if (row.snapshot) {
      pv = penalty_R(ctx, b, s, row.snapshot);
      err = error_norm(std::vector<double>(row.snapshot, row.snapshot + b.n), b.f_true);
    }
    out << row.outer_k << ',' << row.inner_i << ',' << fmt(row.rec.res_data) << ',' << fmt(row.rec.res_damped)
        << ',' << fmt(row.rec.s2_value) << ',' << fmt(row.rec.anorm_est) << ',' << fmt(row.rec.cond_est) << ','
        << fmt(pv) << ',' << fmt(err) << '\n';
  }
}

void write_field(const fs::path& path, const Bundle& b, const char* header, const double* f, bool with_truth) {
  std::ofstream out(path);  // runner.cpp:75-95 / 97-121
  out << header;
  if (b.dims == 1) {
    for (size_t i = 0; i < b.nx; ++i) {
      out << fmt((static_cast<double>(i) + 0.5) * b.h) << ',' << fmt(f[i]);
      if (with_truth) out << ',' << fmt(b.f_true[i]);
      out << '\n';
    }
  } else {
    for (size_t iy = 0; iy < b.ny; ++iy)
      for (size_t ix = 0; ix < b.nx; ++ix) {
        const size_t idx = iy * b.nx + ix;
        out << fmt((static_cast<double>(ix) + 0.5) * b.h) << ','
            << fmt((static_cast<double>(iy) + 0.5) / static_cast<double>(b.ny)) << ',' << fmt(f[idx]);
        if (with_truth) out << ',' << fmt(b.f_true[idx]);
        out << '\n';
      }
  }
}

void write_solution(const fs::path& path, const Bundle& b, const double* f) {
  write_field(path, b, b.dims == 1 ? "x,f,f_true\n" : "x,y,f,f_true\n", f, true);
}

struct RunSummary {  // runner.hpp:14-26
  std::string method;
  int inner_iterations = 0, outer_iterations = 0, iterations_to_discrepancy = -1;
  double final_residual = 0, final_residual_weighted = 0, final_error = 0, final_error_weighted = 0,
         final_penalty = 0;
  std::string stop_reason;
  double wall_seconds = 0;
};

// run_experiment (runner.cpp:134-328) on the device
RunSummary run_experiment(const ExperimentConfig& cfg, const fs::path& out_override,
                          std::optional<uint64_t> seed_override, bool quiet) {
  const auto t0 = std::chrono::steady_clock::now();
  const fs::path out_dir = out_override.empty() ? fs::path(cfg.output.directory) : out_override;
  fs::create_directories(out_dir);
  Ctx ctx;
  Bundle b;
  const uint64_t seed = seed_override.value_or(cfg.problem.seed);
  build_bundle(ctx, cfg.problem, seed, b);
  const SolverConfig& s = cfg.solver;

  // function-space noise level -> Euclidean (runner.cpp:146-151)
  const double sqrt_measure = std::sqrt(b.data_cell_measure);
  mlsqr_stop stop = s.stopping;
  const double delta_euclid = stop.use_s4 ? stop.delta / sqrt_measure : 0.0;
  stop.delta = delta_euclid;
  const bool snaps = cfg.output.traces;  // SolveOptions::record_snapshots (runner.cpp:153-155)

  std::vector<double> solution;
  std::vector<TraceRow> rows;
  std::string stop_reason;
  std::vector<std::string> inner_stop_reasons;
  std::vector<double> eps_used;
  int inner_total = 0, outer_count = 0;
  std::vector<Solve> solves;          // keeps the snapshots alive for the trace rows
  std::vector<std::vector<double>> outer_iterates;
  const std::vector<double> zeros(b.n, 0.0);
  const int holder_levels = s.spd_mode == SpdMode::vcycle ? s.mg_levels : 1;

  switch (s.method) {
    case Method::lsqr:
      solves.push_back(run_krylov(b, nullptr, s.tau, stop, snaps, false));
      break;
    case Method::mlsqr: {
      Pc m, owned;
      eps_used.push_back(assemble_m(ctx, b, s, s.regularizer == "ideal" ? b.f_true : zeros, s.epsilon,
                                    holder_levels, m));
      solves.push_back(run_krylov(b, spd_solver(s, m, owned), s.tau, stop, snaps, false));
      break;
    }
    case Method::cg_normal: {
      Pc m;
      eps_used.push_back(assemble_m(ctx, b, s, s.regularizer == "ideal" ? b.f_true : zeros, s.epsilon, 1, m));
      solves.push_back(run_krylov(b, m.h, s.tau, stop, snaps, true));
      break;
    }
    case Method::lagged_diffusivity: {
      // solve_nonlinear (outer.cpp:40-100), one device solve per outer step
      mlsqr_stop inner = stop;
      inner.max_iters = std::min(inner.max_iters, s.inner_cap);
      std::vector<double> prev(b.n, 0.0), history;
      stop_reason = "max_outer";
      for (int k = 1; k <= s.max_outer; ++k) {
        Pc m, owned;
        // (the reference's lagged branch leaves derived.epsilon_used empty, runner.cpp:186-201)
        assemble_m(ctx, b, s, prev, s.epsilon, holder_levels, m);
        Solve r = run_krylov(b, spd_solver(s, m, owned), s.tau, inner, snaps, false);
        const double pv = penalty_R(ctx, b, s, r.f.data());
        history.push_back(pv);
        ++outer_count;
        inner_total += r.info.iterations;
        inner_stop_reasons.emplace_back(stop_name(r.info.stop_reason));
        if (cfg.output.outer_snapshots) outer_iterates.push_back(r.f);
        std::vector<double> cur = r.f;
        solves.push_back(std::move(r));
        bool stagnated = false;  // outer_stop_check (outer.cpp:31-38)
        if (history.size() >= 2) {
          const double pr = history[history.size() - 2];
          stagnated = pr == 0.0 || (history.back() - pr) / pr > -s.rel_decrease_threshold;
        }
        if (stagnated) {
          stop_reason = "stagnation";
          break;
        }
        prev = std::move(cur);
      }
      solution = prev;
      break;
    }
  }
  if (s.method != Method::lagged_diffusivity) {
    solution = solves[0].f;
    stop_reason = stop_name(solves[0].info.stop_reason);
    inner_total = solves[0].info.iterations;
  }
  for (size_t k = 0; k < solves.size(); ++k) {
    const Solve& r = solves[k];
    const int outer_k = s.method == Method::lagged_diffusivity ? static_cast<int>(k) + 1 : 0;
    for (size_t i = 0; i < r.trace.size(); ++i)
      rows.push_back({outer_k, static_cast<int>(i) + 1, r.trace[i],
                      i * b.n < r.snaps.size() ? r.snaps.data() + i * b.n : nullptr});
  }

  if (cfg.output.traces) write_trace(ctx, out_dir / "trace.csv", rows, b, s);
  if (cfg.output.solutions) write_solution(out_dir / "solution.csv", b, solution.data());

  if (cfg.output.basis_vectors > 0) {  // runner.cpp:245-275
    const int k = cfg.output.basis_vectors;
    std::vector<double> vec((size_t)k * b.n);
    int count = 0, exhausted = 0;
    if (s.method == Method::mlsqr || s.method == Method::lagged_diffusivity) {
      // priorconditioned space, always with the exact factorization (runner.cpp:252-263)
      Pc m, chol;
      const std::vector<double>& field =
          s.method == Method::mlsqr ? (s.regularizer == "ideal" ? b.f_true : zeros) : solution;
      assemble_m(ctx, b, s, field, s.epsilon, 1, m);
      check(mlsqr_chol_map_create(m.h, &chol.h, nullptr));
      check(mlsqr_krylov_basis(b.op.h, chol.h, nullptr, s.tau, b.g.data(), k, vec.data(), &count, &exhausted,
                               MLSQR_HOST));
    } else if (s.method == Method::cg_normal) {
      Pc m;
      assemble_m(ctx, b, s, s.regularizer == "ideal" ? b.f_true : zeros, s.epsilon, 1, m);
      check(mlsqr_krylov_basis(b.op.h, nullptr, m.h, s.tau, b.g.data(), k, vec.data(), &count, &exhausted,
                               MLSQR_HOST));
    } else if (s.tau > 0.0) {
      // SparseSpd::identity: a holder with no edges and unit shift is I
      Pc m;
      check(mlsqr_vcycle_create(ctx.h, b.dims, b.nx, b.ny, 1, b.h, 1, 1, 1, 1.0, 1, &m.h));
      check(mlsqr_vcycle_set_coefficients(m.h, zeros.data(), b.dims >= 2 ? zeros.data() : nullptr, nullptr, 1.0,
                                          MLSQR_HOST));
      check(mlsqr_krylov_basis(b.op.h, nullptr, m.h, s.tau, b.g.data(), k, vec.data(), &count, &exhausted,
                               MLSQR_HOST));
    } else {
      check(mlsqr_krylov_basis(b.op.h, nullptr, nullptr, 0.0, b.g.data(), k, vec.data(), &count, &exhausted,
                               MLSQR_HOST));
    }
    for (int j = 0; j < count; ++j) {  // write_basis (runner.cpp:97-121)
      char name[32];
      std::snprintf(name, sizeof name, "basis_%03d.csv", j);
      write_field(out_dir / name, b, b.dims == 1 ? "x,v\n" : "x,y,v\n", vec.data() + (size_t)j * b.n, false);
    }
  }
  if (cfg.output.outer_snapshots && s.method == Method::lagged_diffusivity) {
    for (size_t k = 0; k < outer_iterates.size(); ++k) {
      char name[40];
      std::snprintf(name, sizeof name, "solution_outer_%03d.csv", static_cast<int>(k) + 1);
      write_solution(out_dir / name, b, outer_iterates[k].data());
    }
  }

  RunSummary sum;
  sum.method = method_name(s.method);
  sum.inner_iterations = inner_total;
  sum.outer_iterations = outer_count;
  if (stop.use_s4) {  // first_discrepancy_row (runner.cpp:123-130)
    for (size_t i = 0; i < rows.size(); ++i)
      if (rows[i].rec.res_data <= stop.eta * delta_euclid) {
        sum.iterations_to_discrepancy = static_cast<int>(i) + 1;
        break;
      }
  }
  {
    std::vector<double> af(b.n);
    check(mlsqr_op_apply(b.op.h, solution.data(), b.n, af.data(), b.n, MLSQR_HOST));
    double acc = 0.0;
    for (size_t i = 0; i < b.n; ++i) {
      const double d = b.g[i] - af[i];
      acc += d * d;
    }
    sum.final_residual = std::sqrt(acc);
  }
  sum.final_residual_weighted = sqrt_measure * sum.final_residual;
  sum.final_error = error_norm(solution, b.f_true);
  sum.final_error_weighted = std::sqrt(b.data_cell_measure) * sum.final_error;
  sum.final_penalty = penalty_R(ctx, b, s, solution.data());
  sum.stop_reason = stop_reason;
  sum.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  json meta;  // runner.cpp:301-325
  meta["config"] = {{"problem", cfg.problem.raw},
                    {"method", sum.method},
                    {"tau", s.tau},
                    {"seed_used", seed}};
  meta["derived"] = {{"data_cell_measure", b.data_cell_measure},
                     {"delta_euclid", delta_euclid},
                     {"epsilon_used", eps_used},
                     {"kernels_backend", std::string(mlsqr_version())}};
  meta["result"] = {{"stop_reason", sum.stop_reason},
                    {"inner_stop_reasons", inner_stop_reasons},
                    {"inner_iterations", sum.inner_iterations},
                    {"outer_iterations", sum.outer_iterations},
                    {"iterations_to_discrepancy", sum.iterations_to_discrepancy},
                    {"final_residual", sum.final_residual},
                    {"final_residual_weighted", sum.final_residual_weighted},
                    {"final_error", sum.final_error},
                    {"final_error_weighted", sum.final_error_weighted},
                    {"final_penalty", sum.final_penalty}};
  meta["wall_seconds"] = sum.wall_seconds;
  meta["timestamp"] = std::chrono::duration_cast<std::chrono::milliseconds>(
                          std::chrono::system_clock::now().time_since_epoch())
                          .count();
  std::ofstream meta_out(out_dir / "meta.json");
  meta_out << meta.dump(2) << '\n';

  if (!quiet) {
    std::cout << sum.method << ": " << sum.inner_iterations << " iterations";
    if (outer_count > 0) std::cout << " over " << outer_count << " outer steps";
    std::cout << ", stop=" << sum.stop_reason << ", residual=" << sum.final_residual_weighted
              << " (weighted), error=" << sum.final_error << '\n'
              << "artifacts in " << out_dir.string() << '\n';
  }
  return sum;
}

// compare_experiments (runner.cpp:330-366)
void compare_experiments(const ExperimentConfig& a, const ExperimentConfig& b, const fs::path& out_root,
                         std::optional<uint64_t> seed, bool quiet) {
  if (a.problem.raw != b.problem.raw) throw ConfigError("compare requires identical problem sections");
  const fs::path root = out_root.empty() ? fs::path("compare_out") : out_root;
  const RunSummary sa = run_experiment(a, root / "a", seed, true);
  const RunSummary sb = run_experiment(b, root / "b", seed, true);
  if (quiet) return;
  auto line = [](const std::string& name, const std::string& va, const std::string& vb) {
    std::printf("%-28s %20s %20s\n", name.c_str(), va.c_str(), vb.c_str());
  };
  line("metric", sa.method, sb.method);
  line("iterations_to_discrepancy", std::to_string(sa.iterations_to_discrepancy),
       std::to_string(sb.iterations_to_discrepancy));
  line("inner_iterations", std::to_string(sa.inner_iterations), std::to_string(sb.inner_iterations));
  line("final_error", fmt(sa.final_error), fmt(sb.final_error));
  line("final_penalty", fmt(sa.final_penalty), fmt(sb.final_penalty));
  line("final_residual_weighted", fmt(sa.final_residual_weighted), fmt(sb.final_residual_weighted));
  line("stop_reason", sa.stop_reason, sb.stop_reason);
}

// exit codes (tools/main.cpp:13-16): 0 ok, 2 usage / missing file, 3 config schema violation,
// 4 solver breakdown, 1 anything else
constexpr int kExitUsage = 2, kExitConfig = 3, kExitSolver = 4;

int usage(const char* prog) {
  std::cerr << "usage: " << prog << " [--out DIR] [--seed N] [--quiet] run CONFIG\n"
            << "       " << prog << " [--out DIR] [--seed N] [--quiet] compare CONFIG_A CONFIG_B\n";
  return kExitUsage;
}

}  // namespace

int main(int argc, char** argv) {
  std::string out_dir;
  std::optional<uint64_t> seed;
  bool quiet = false;
  std::vector<std::string> pos;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--out" && i + 1 < argc) out_dir = argv[++i];
    else if (a == "--seed" && i + 1 < argc) {
      try {
        seed = std::stoull(argv[++i]);
      } catch (...) {
        return usage(argv[0]);
      }
    } else if (a == "--quiet") quiet = true;
    else if (a == "-h" || a == "--help") {
      usage(argv[0]);
      return 0;
    } else if (!a.empty() && a[0] == '-') return usage(argv[0]);
    else pos.push_back(a);
  }
  const bool run = pos.size() == 2 && pos[0] == "run", cmp = pos.size() == 3 && pos[0] == "compare";
  if (!run && !cmp) return usage(argv[0]);
  for (size_t i = 1; i < pos.size(); ++i) {
    if (!fs::exists(pos[i])) {
      std::cerr << "error: config file not found: " << pos[i] << '\n';
      return kExitUsage;
    }
  }
  try {
    if (run) run_experiment(load_config(pos[1]), out_dir, seed, quiet);
    else compare_experiments(load_config(pos[1]), load_config(pos[2]), out_dir, seed, quiet);
  } catch (const ConfigError& e) {
    std::cerr << "config error: " << e.what() << '\n';
    return kExitConfig;
  } catch (const SolverFailure& e) {
    std::cerr << "solver breakdown: " << e.what() << '\n';
    return kExitSolver;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
  return 0;
}
