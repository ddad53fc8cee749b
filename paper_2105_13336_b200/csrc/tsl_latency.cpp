// Cold-start latency predictor: LatencyPredictor (latency.hpp:45-66;
// latency.cpp:11-135) and predict_latencies (orchestrator.cpp:72-87), the
// latency source of Orchestrator::plan_cold_start. Host code around the
// device planner: per op kind, a least-squares fit of
//   latency ~ features + usage^2 + intercept
// solved for the minimum-norm solution (what the reference's Eigen
// completeOrthogonalDecomposition().solve computes) by a one-sided Jacobi SVD
// of the small design matrix, singular values below eps * max(m, n) * s_max
// treated as zero. JSON I/O writes the reference's ordered_json dump(2).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "tensile_b200.h"
#include "tsl_graph.h"

using namespace tsl::hostg;

struct tsl_predictor {
  struct Model {
    std::vector<double> coef;  // one per feature value + the usage^2 term
    double intercept = 0.0;
    double r2 = 0.0;
  };
  std::map<std::string, Model> models;
};

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return TSL_OK;
  } catch (const Fail& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TSL_ERR_INTERNAL;
  }
}

// Minimum-norm least squares x = pinv(A) b, A row-major m x n (one-sided
// Jacobi: orthogonalize A's columns by plane rotations accumulated in V;
// then A V = U S and x = V S^+ U^T b).
std::vector<double> min_norm_lstsq(std::vector<double> A, const std::vector<double>& b, int m, int n) {
  std::vector<double> V(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) V[size_t(i) * n + i] = 1.0;
  auto col = [&](int j, int r) -> double& { return A[size_t(r) * n + j]; };
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int r = 0; r < m; ++r) {
          alpha += col(p, r) * col(p, r);
          beta += col(q, r) * col(q, r);
          gamma += col(p, r) * col(q, r);
        }
        if (gamma == 0.0 || std::abs(gamma) <= eps * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = std::copysign(1.0, zeta) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int r = 0; r < m; ++r) {
          const double ap = col(p, r), aq = col(q, r);
          col(p, r) = c * ap - s * aq;
          col(q, r) = s * ap + c * aq;
        }
        for (int r = 0; r < n; ++r) {
          const double vp = V[size_t(r) * n + p], vq = V[size_t(r) * n + q];
          V[size_t(r) * n + p] = c * vp - s * vq;
          V[size_t(r) * n + q] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> sigma(n, 0.0);
  double smax = 0.0;
  for (int j = 0; j < n; ++j) {
    double ss = 0;
    for (int r = 0; r < m; ++r) ss += col(j, r) * col(j, r);
    sigma[j] = std::sqrt(ss);
    smax = std::max(smax, sigma[j]);
  }
  const double thr = eps * double(std::max(m, n)) * smax;
  std::vector<double> x(n, 0.0);
  for (int j = 0; j < n; ++j) {
    if (!(sigma[j] > thr)) continue;
    double ub = 0;  // (u_j . b) / s_j with u_j = A[:, j] / s_j
    for (int r = 0; r < m; ++r) ub += col(j, r) * b[r];
    const double w = ub / (sigma[j] * sigma[j]);
    for (int i = 0; i < n; ++i) x[i] += V[size_t(i) * n + j] * w;
  }
  return x;
}

// nlohmann::json's number text for a double (shortest round trip; fixed
// notation for decimal exponents in (-4, 15], else d.ddde+XX; ".0" on
// integral values; NaN / infinity print null).
std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  std::string s(buf, r.ptr);
  std::string sign;
  if (s[0] == '-') { sign = "-"; s = s.substr(1); }
  const size_t epos = s.find('e');
  std::string digits = s.substr(0, epos);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int e10 = std::stoi(s.substr(epos + 1));
  const int len = int(digits.size());
  const int k = e10 - (len - 1);  // value = digits * 10^k
  const int n = len + k;          // decimal point position
  std::string o;
  if (k >= 0 && n <= 15) {
    o = digits + std::string(k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    o = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    o = "0." + std::string(-n, '0') + digits;
  } else {
    const int e = n - 1;
    o = digits.substr(0, 1);
    if (len > 1) o += "." + digits.substr(1);
    o += e < 0 ? "e-" : "e+";
    const int ae = std::abs(e);
    o += ae < 10 ? "0" + std::to_string(ae) : std::to_string(ae);
  }
  return sign + o;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') { o += '\\'; o += c; }
    else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else o += c;
  }
  return o + "\"";
}

// A minimal reader for the predictor document (an object of objects with
// "coefficients": [numbers], "intercept": number, "r2": number).
struct Reader {
  const char* p;
  void ws() { while (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t') ++p; }
  void expect(char c) {
    ws();
    if (*p != c) fail(TSL_ERR_VALIDATION, std::string("predictor JSON: expected '") + c + "'");
    ++p;
  }
  bool peek(char c) { ws(); return *p == c; }
  std::string str() {
    expect('"');
    std::string o;
    while (*p && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (*p == 'u') {
          o += char(std::strtol(std::string(p + 1, 4).c_str(), nullptr, 16));
          p += 5;
          continue;
        }
      }
      o += *p++;
    }
    expect('"');
    return o;
  }
  double number() {
    ws();
    if (std::strncmp(p, "null", 4) == 0) { p += 4; return std::numeric_limits<double>::quiet_NaN(); }
    char* end = nullptr;
    const double v = std::strtod(p, &end);
    if (end == p) fail(TSL_ERR_VALIDATION, "predictor JSON: expected a number");
    p = end;
    return v;
  }
};

}  // namespace

extern "C" {

// LatencyPredictor::fit (latency.cpp:79-126): samples k have op kind
// op_kinds[k], feature values values[value_offsets[k] .. value_offsets[k+1])
// (input dims, attributes, gpu usage last) and label labels[k].
int tsl_latency_fit(int32_t n, const char* const* op_kinds, const int32_t* value_offsets, const double* values,
                    const double* labels, tsl_predictor** out) {
  if (!out || n < 0 || (n > 0 && (!op_kinds || !value_offsets || !values || !labels))) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    std::map<std::string, std::vector<int32_t>> by_kind;
    for (int32_t k = 0; k < n; ++k) by_kind[op_kinds[k] ? op_kinds[k] : ""].push_back(k);
    auto p = std::make_unique<tsl_predictor>();
    for (const auto& [kind, rows] : by_kind) {
      if (rows.size() < 2) fail(TSL_ERR_VALIDATION, "insufficient samples for op kind " + kind);
      const int32_t width = value_offsets[rows[0] + 1] - value_offsets[rows[0]];
      for (int32_t r : rows)
        if (value_offsets[r + 1] - value_offsets[r] != width)
          fail(TSL_ERR_VALIDATION, "inconsistent feature width for op kind " + kind);
      bool degenerate = true;
      for (int32_t r : rows)
        if (!std::equal(values + value_offsets[r], values + value_offsets[r + 1], values + value_offsets[rows[0]]))
          degenerate = false;
      if (degenerate) fail(TSL_ERR_VALIDATION, "degenerate (all-identical) features for op kind " + kind);
      // design matrix: features, usage^2, intercept column
      const int m = int(rows.size()), nc = width + 2;
      std::vector<double> X(size_t(m) * nc), y(m);
      for (int i = 0; i < m; ++i) {
        const double* v = values + value_offsets[rows[i]];
        for (int c = 0; c < width; ++c) X[size_t(i) * nc + c] = v[c];
        const double u = width > 0 ? v[width - 1] : 0.0;
        X[size_t(i) * nc + width] = u * u;
        X[size_t(i) * nc + width + 1] = 1.0;
        y[i] = labels[rows[i]];
      }
      const std::vector<double> beta = min_norm_lstsq(X, y, m, nc);
      tsl_predictor::Model md;
      md.coef.assign(beta.begin(), beta.begin() + width + 1);
      md.intercept = beta[width + 1];
      double mean = 0;
      for (double v : y) mean += v;
      mean /= m;
      double ss_tot = 0, ss_res = 0;
      for (int i = 0; i < m; ++i) {
        double f = 0;
        for (int c = 0; c < nc; ++c) f += X[size_t(i) * nc + c] * beta[c];
        ss_tot += (y[i] - mean) * (y[i] - mean);
        ss_res += (y[i] - f) * (y[i] - f);
      }
      md.r2 = ss_tot > 0.0 ? 1.0 - ss_res / ss_tot : 1.0;
      p->models[kind] = std::move(md);
    }
    *out = p.release();
  });
}

void tsl_latency_destroy(tsl_predictor* p) { delete p; }

// LatencyPredictor::to_json (latency.cpp:128-135): nlohmann ordered_json dump(2) + "\n".
char* tsl_latency_to_json(const tsl_predictor* p) {
  if (!p) return nullptr;
  std::string o;
  if (p->models.empty()) {
    o = "{}\n";
  } else {
    o = "{\n";
    bool first = true;
    for (const auto& [kind, m] : p->models) {
      if (!first) o += ",\n";
      first = false;
      o += "  " + jstr(kind) + ": {\n    \"coefficients\": ";
      if (m.coef.empty()) {
        o += "[]";
      } else {
        o += "[\n";
        for (size_t i = 0; i < m.coef.size(); ++i) o += "      " + num(m.coef[i]) + (i + 1 < m.coef.size() ? ",\n" : "\n");
        o += "    ]";
      }
      o += ",\n    \"intercept\": " + num(m.intercept) + ",\n    \"r2\": " + num(m.r2) + "\n  }";
    }
    o += "\n}\n";
  }
  char* s = static_cast<char*>(std::malloc(o.size() + 1));
  std::memcpy(s, o.c_str(), o.size() + 1);
  return s;
}

// LatencyPredictor::from_json (latency.cpp:137-149).
int tsl_latency_from_json(const char* doc, tsl_predictor** out) {
  if (!doc || !out) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    auto p = std::make_unique<tsl_predictor>();
    Reader r{doc};
    r.expect('{');
    while (!r.peek('}')) {
      const std::string kind = r.str();
      r.expect(':');
      r.expect('{');
      tsl_predictor::Model m;
      bool hc = false, hi = false, hr = false;
      while (!r.peek('}')) {
        const std::string key = r.str();
        r.expect(':');
        if (key == "coefficients") {
          hc = true;
          r.expect('[');
          while (!r.peek(']')) {
            m.coef.push_back(r.number());
            if (r.peek(',')) r.expect(',');
          }
          r.expect(']');
        } else if (key == "intercept") {
          hi = true;
          m.intercept = r.number();
        } else if (key == "r2") {
          hr = true;
          m.r2 = r.number();
        } else {
          r.number();
        }
        if (r.peek(',')) r.expect(',');
      }
      r.expect('}');
      if (!hc) fail(TSL_ERR_VALIDATION, "[json.exception.out_of_range.403] key 'coefficients' not found");
      if (!hi) fail(TSL_ERR_VALIDATION, "[json.exception.out_of_range.403] key 'intercept' not found");
      if (!hr) fail(TSL_ERR_VALIDATION, "[json.exception.out_of_range.403] key 'r2' not found");
      p->models[kind] = std::move(m);
      if (r.peek(',')) r.expect(',');
    }
    r.expect('}');
    *out = p.release();
  });
}

// LatencyPredictor::predict (latency.cpp:54-68), clamped at zero.
int tsl_latency_predict(const tsl_predictor* p, const char* op_kind, const double* values, int32_t n, double* out) {
  if (!p || !op_kind || !out || (n > 0 && !values)) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    auto it = p->models.find(op_kind);
    if (it == p->models.end()) fail(TSL_ERR_VALIDATION, std::string("no fitted model for op kind ") + op_kind);
    const auto& m = it->second;
    if (int32_t(m.coef.size()) != n + 1)
      fail(TSL_ERR_VALIDATION, std::string("feature width mismatch for op kind ") + op_kind);
    double y = m.intercept;
    for (int32_t i = 0; i < n; ++i) y += m.coef[i] * values[i];
    const double usage = n > 0 ? values[n - 1] : 0.0;
    y += m.coef.back() * usage * usage;
    *out = std::max(0.0, y);
  });
}

int tsl_latency_r2(const tsl_predictor* p, const char* op_kind, double* out) {
  if (!p || !op_kind || !out) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    auto it = p->models.find(op_kind);
    if (it == p->models.end()) fail(TSL_ERR_VALIDATION, std::string("no fitted model for op kind ") + op_kind);
    *out = it->second.r2;
  });
}

// predict_latencies (orchestrator.cpp:72-87): every op's latency from its
// kind's model -- features = each input tensor's size (one slot per input,
// derive_layouts width), the op's attributes, then gpu_usage -- rounded to
// ticks. Attributes: op_attr_offsets[n_ops+1] into op_attrs (NULL: none).
int tsl_predict_latencies(const tsl_predictor* p, const tsl_job_desc* job, const int32_t* op_attr_offsets,
                          const double* op_attrs, double gpu_usage, int64_t* out) {
  if (!p || !job || !out) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    const int32_t O = job->n_ops;
    auto nattr = [&](int32_t o) { return op_attr_offsets ? op_attr_offsets[o + 1] - op_attr_offsets[o] : 0; };
    // derive_layouts (latency.cpp:42-52): per kind, the widest op
    std::map<std::string, std::pair<int32_t, int32_t>> layout;
    for (int32_t o = 0; o < O; ++o) {
      auto& l = layout[job->op_kinds[o] ? job->op_kinds[o] : ""];
      l.first = std::max(l.first, job->op_in_offsets[o + 1] - job->op_in_offsets[o]);
      l.second = std::max(l.second, nattr(o));
    }
    std::vector<double> fv;
    for (int32_t o = 0; o < O; ++o) {
      const std::string kind = job->op_kinds[o] ? job->op_kinds[o] : "";
      const auto& l = layout.at(kind);
      // extract_features (latency.cpp:11-40)
      if (gpu_usage < 0.0 || gpu_usage > 1.0) {
        char b[64];
        std::snprintf(b, sizeof b, "%f", gpu_usage);
        fail(TSL_ERR_VALIDATION, std::string("gpu_usage out of [0,1]: ") + b);
      }
      fv.assign(size_t(l.first) + l.second + 1, 0.0);
      int32_t slot = 0;
      for (int32_t i = job->op_in_offsets[o]; i < job->op_in_offsets[o + 1]; ++i) {
        if (slot >= l.first) fail(TSL_ERR_VALIDATION, std::string("feature layout too narrow for op ") + job->op_ids[o]);
        fv[slot++] = double(job->tensor_sizes[job->op_inputs[i]]);
      }
      for (int32_t a = 0; a < nattr(o); ++a) fv[size_t(l.first) + a] = op_attrs[op_attr_offsets[o] + a];
      fv.back() = gpu_usage;
      double y = 0;
      const int rc = tsl_latency_predict(p, kind.c_str(), fv.data(), int32_t(fv.size()), &y);
      if (rc) fail(rc, tsl_last_error());
      out[o] = int64_t(std::llround(y));
    }
  });
}

}  // extern "C"
