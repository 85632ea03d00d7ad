// Results writer (output side): the files of the
// reference's write_results (P:src/io.cpp:571-720), written in parallel.
// Rows are formatted by all host threads into per-task buffers, then
// pwrite()n at their prefix-summed offsets.  The numbers are formatted with
// std::to_chars(general, 17), which is exact and prints the same characters
// as the reference's fmt17 "%.17g" (io.cpp:25-29).  The device has already
// reduced the accumulators (diag kernels), so this file only formats.
#include "output_host.h"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <thread>
#include <vector>

namespace cmc {
namespace {

namespace fs = std::filesystem;

void set_err(cmc_error* err, int code, const std::string& msg) {
  if (!err) return;
  std::memset(err, 0, sizeof(*err));
  err->code = code;
  err->index1 = err->index2 = -1;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
}

int n_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? (int)hw : 1;
}

template <class F>
void run_threads(int T, F&& body) {
  if (T <= 1) {
    body(0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back([&body, t] { body(t); });
  for (auto& x : th) x.join();
}

// fmt17 (io.cpp:25-29): "%.17g"
inline void put17(std::string& out, double v) {
  char buf[40];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
  out.append(buf, r.ptr);
}

inline void put_long(std::string& out, long long v) {
  char buf[24];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, r.ptr);
}

// csv_escape (io.cpp:32-44)
void put_csv(std::string& out, const char* s) {
  if (!std::strchr(s, ',') && !std::strchr(s, '"')) {
    out.append(s);
    return;
  }
  out.push_back('"');
  for (const char* p = s; *p; ++p) {
    if (*p == '"') out.push_back('"');
    out.push_back(*p);
  }
  out.push_back('"');
}

// A file written by parallel tasks: rows [0, n) are cut into tasks of
// `chunk` rows, formatted by T threads, and pwrite()n in order.
class RowFile {
 public:
  RowFile(const std::string& path) : path_(path) {
    fd_ = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  }
  ~RowFile() {
    if (fd_ >= 0) ::close(fd_);
  }
  bool ok() const { return fd_ >= 0 && !failed_; }

  void put(const std::string& s) {
    if (!write_at(s.data(), s.size(), off_)) failed_ = true;
    off_ += (off_t)s.size();
  }

  template <class Fmt>
  void rows(long n, long chunk, Fmt&& fmt) {
    const int T = n_threads();
    const long tasks = (n + chunk - 1) / chunk;
    for (long t0 = 0; t0 < tasks && !failed_; t0 += 4L * T) {
      const long nt = std::min<long>(4L * T, tasks - t0);
      std::vector<std::string> bufs((size_t)nt);
      run_threads(std::min<long>(T, nt), [&](int t) {
        for (long k = t; k < nt; k += T) {
          const long r0 = (t0 + k) * chunk, r1 = std::min(n, r0 + chunk);
          std::string& b = bufs[(size_t)k];
          b.reserve((size_t)(r1 - r0) * 64);
          for (long r = r0; r < r1; ++r) fmt(r, b);
        }
      });
      std::vector<off_t> at((size_t)nt);
      for (long k = 0; k < nt; ++k) {
        at[(size_t)k] = off_;
        off_ += (off_t)bufs[(size_t)k].size();
      }
      std::vector<char> bad((size_t)nt, 0);
      run_threads(std::min<long>(T, nt), [&](int t) {
        for (long k = t; k < nt; k += T)
          if (!write_at(bufs[(size_t)k].data(), bufs[(size_t)k].size(), at[(size_t)k]))
            bad[(size_t)k] = 1;
      });
      for (char b : bad) failed_ |= b != 0;
    }
  }

 private:
  bool write_at(const char* p, size_t n, off_t at) {
    while (n > 0) {
      const ssize_t w = ::pwrite(fd_, p, n, at);
      if (w <= 0) return false;
      p += w;
      n -= (size_t)w;
      at += w;
    }
    return true;
  }
  std::string path_;
  int fd_ = -1;
  off_t off_ = 0;
  bool failed_ = false;
};

// ensure_writable (io.cpp:467-480)
int ensure_writable(const std::string& outdir, cmc_error* err) {
  std::error_code ec;
  fs::create_directories(fs::path(outdir) / "samples", ec);
  if (ec) {
    set_err(err, CMC_ERR_CONFIG,
            "cannot create output directory '" + outdir + "': " + ec.message());
    return CMC_ERR_CONFIG;
  }
  const fs::path probe = fs::path(outdir) / ".write_probe";
  {
    std::ofstream out(probe);
    if (!out) {
      set_err(err, CMC_ERR_CONFIG, "output directory '" + outdir + "' is not writable");
      return CMC_ERR_CONFIG;
    }
    out << "ok";
  }
  fs::remove(probe, ec);
  return CMC_OK;
}

int cannot_write(const std::string& path, cmc_error* err) {
  set_err(err, CMC_ERR_CONFIG, "cannot write file '" + path + "'");
  return CMC_ERR_CONFIG;
}

// ---- run_report.json in nlohmann::json dump(2) layout (sorted keys) ----

// nlohmann's number_float output: shortest round-trip digits, placed by
// format_buffer(min_exp = -4, max_exp = 15).
void json_double(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (v == 0.0) {
    out += std::signbit(v) ? "-0.0" : "0.0";
    return;
  }
  char sci[40];
  const auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
  *r.ptr = 0;
  const char* p = sci;
  if (*p == '-') {
    out.push_back('-');
    ++p;
  }
  std::string digits;
  for (; *p && *p != 'e'; ++p)
    if (*p != '.') digits.push_back(*p);
  const int e10 = std::atoi(p + 1);  // value = d.ddd * 10^e10
  const int k = (int)digits.size();
  const int n = e10 + 1;  // decimal point position
  if (k <= n && n <= 15) {
    out += digits;
    out.append((size_t)(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= 15) {
    out.append(digits, 0, (size_t)n);
    out.push_back('.');
    out.append(digits, (size_t)n, std::string::npos);
  } else if (-4 < n && n <= 0) {
    out += "0.";
    out.append((size_t)(-n), '0');
    out += digits;
  } else {
    out.push_back(digits[0]);
    if (k > 1) {
      out.push_back('.');
      out.append(digits, 1, std::string::npos);
    }
    out.push_back('e');
    const int ex = n - 1;
    out.push_back(ex < 0 ? '-' : '+');
    const int a = std::abs(ex);
    if (a < 10) out.push_back('0');
    out += std::to_string(a);
  }
}

struct Json {
  // minimal ordered tree: objects keep keys sorted like std::map
  enum Kind { INT, UINT, DBL, STR, ARR, OBJ } kind = OBJ;
  long long i = 0;
  unsigned long long u = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  static Json I(long long v) { Json j; j.kind = INT; j.i = v; return j; }
  static Json U(unsigned long long v) { Json j; j.kind = UINT; j.u = v; return j; }
  static Json D(double v) { Json j; j.kind = DBL; j.d = v; return j; }
  static Json S(const std::string& v) { Json j; j.kind = STR; j.s = v; return j; }
  static Json A() { Json j; j.kind = ARR; return j; }
  Json& set(const std::string& k, Json v) {
    auto it = std::lower_bound(obj.begin(), obj.end(), k,
                               [](const auto& a, const std::string& b) { return a.first < b; });
    return obj.insert(it, {k, std::move(v)})->second;
  }

  void dump(std::string& out, int depth) const {
    const std::string ind((size_t)(2 * (depth + 1)), ' '), end((size_t)(2 * depth), ' ');
    switch (kind) {
      case INT: out += std::to_string(i); break;
      case UINT: out += std::to_string(u); break;
      case DBL: json_double(out, d); break;
      case STR:
        out.push_back('"');
        for (char c : s) {
          if (c == '"' || c == '\\') out.push_back('\\');
          out.push_back(c);
        }
        out.push_back('"');
        break;
      case ARR:
        if (arr.empty()) {
          out += "[]";
          break;
        }
        out += "[\n";
        for (size_t k = 0; k < arr.size(); ++k) {
          out += ind;
          arr[k].dump(out, depth + 1);
          out += k + 1 < arr.size() ? ",\n" : "\n";
        }
        out += end + "]";
        break;
      case OBJ:
        if (obj.empty()) {
          out += "{}";
          break;
        }
        out += "{\n";
        for (size_t k = 0; k < obj.size(); ++k) {
          out += ind + "\"" + obj[k].first + "\": ";
          obj[k].second.dump(out, depth + 1);
          out += k + 1 < obj.size() ? ",\n" : "\n";
        }
        out += end + "}";
        break;
    }
  }
};

const char* kStepNames[7] = {"epsilon", "gamma", "nu", "tau", "beta", "theta", "sigma"};

}  // namespace

int write_results_files(const ResultsInput& in, cmc_error* err) {
  const long C = in.C, G = in.G, L = in.L;
  const double Cd = static_cast<double>(C);
  int rc = ensure_writable(in.outdir, err);
  if (rc) return rc;
  const fs::path root(in.outdir);
  const long beta0 = 2 + 2 * L, gam0 = beta0 + G * L;

  auto put_est = [&](std::string& b, long row) {
    b.push_back(',');
    put17(b, in.mean[(size_t)row]);
    b.push_back(',');
    put17(b, in.sd[(size_t)row]);
    b.push_back(',');
    put17(b, in.lo[(size_t)row]);
    b.push_back(',');
    put17(b, in.hi[(size_t)row]);
  };
  std::vector<long> gene_contrasts, global_contrasts;
  for (size_t k = 0; k < in.contrast_ids.size(); ++k)
    (in.per_gene[k] ? gene_contrasts : global_contrasts).push_back((long)k);

  {  // gene_estimates.csv
    const std::string path = (root / "gene_estimates.csv").string();
    RowFile f(path);
    if (!f.ok()) return cannot_write(path, err);
    std::string h = "gene";
    for (long l = 0; l < L; ++l) {
      const std::string base = "beta[" + std::to_string(l + 1) + "]";
      h += "," + base + "_mean," + base + "_sd," + base + "_lo95," + base + "_hi95";
    }
    h += ",gamma_mean,gamma_sd,gamma_lo95,gamma_hi95";
    for (long k : gene_contrasts) h += ",prob_" + in.contrast_ids[(size_t)k];
    h += '\n';
    f.put(h);
    f.rows(G, 2048, [&](long g, std::string& b) {
      if (in.genes) {
        put_csv(b, in.genes[g]);
      } else {
        b.push_back('g');
        put_long(b, g + 1);
      }
      for (long l = 0; l < L; ++l) put_est(b, beta0 + g * L + l);
      put_est(b, gam0 + g);
      for (long k : gene_contrasts) {
        double p = 0.0;
        for (long c = 0; c < C; ++c)
          p += in.probs[(size_t)(c * in.n_prob + in.prob_off[(size_t)k] + g)];
        b.push_back(',');
        put17(b, p / Cd);
      }
      b.push_back('\n');
    });
    if (!f.ok()) return cannot_write(path, err);
  }

  {  // hyper_estimates.csv
    const std::string path = (root / "hyper_estimates.csv").string();
    RowFile f(path);
    if (!f.ok()) return cannot_write(path, err);
    std::string b = "param,mean,sd,lo95,hi95\n";
    auto named = [&](const std::string& name, long row) {
      b += name;
      put_est(b, row);
      b.push_back('\n');
    };
    named("nu", 0);
    named("tau", 1);
    for (long l = 0; l < L; ++l) named("theta[" + std::to_string(l + 1) + "]", 2 + l);
    for (long l = 0; l < L; ++l) named("sigma[" + std::to_string(l + 1) + "]", 2 + L + l);
    for (long k : global_contrasts) {
      double p = 0.0;
      for (long c = 0; c < C; ++c) p += in.probs[(size_t)(c * in.n_prob + in.prob_off[(size_t)k])];
      p /= Cd;
      // indicator stream: mean of squares equals the mean (io.cpp:637-638);
      // write_estimate + credible_interval (P:src/diagnostics.cpp:46-57)
      double var = p - p * p;
      const double slack = 1e-9 * std::max(1.0, std::fabs(p));
      if (var < -slack) {
        set_err(err, CMC_ERR_CONFIG, "moment accumulator corruption: meansq < mean^2");
        return CMC_ERR_CONFIG;
      }
      const double sdv = std::sqrt(std::max(0.0, p - p * p));
      if (var < 0.0) var = 0.0;
      const double half = in.z * std::sqrt(var);
      b += "contrast[" + in.contrast_ids[(size_t)k] + "]";
      for (double v : {p, sdv, p - half, p + half}) {
        b.push_back(',');
        put17(b, v);
      }
      b.push_back('\n');
    }
    f.put(b);
    if (!f.ok()) return cannot_write(path, err);
  }

  {  // diagnostics.csv
    const std::string path = (root / "diagnostics.csv").string();
    RowFile f(path);
    if (!f.ok()) return cannot_write(path, err);
    f.put("param,rhat,ess,status,pass\n");
    if (in.diag_error) {  // build_diagnostics throws after the header is out
      set_err(err, CMC_ERR_CONFIG, in.diag_error_msg);
      return CMC_ERR_CONFIG;
    }
    const long R = gam0 + G;
    static const char* kEss[3] = {"ok", "undefined", "degenerate"};
    f.rows(R, 8192, [&](long r, std::string& b) {
      if (r < 2) {
        b += r == 0 ? "nu" : "tau";
      } else if (r < beta0) {
        b += r < 2 + L ? "theta[" : "sigma[";
        put_long(b, (r - 2) % L + 1);
        b.push_back(']');
      } else if (r < gam0) {
        b += "\"beta[";  // the comma in the name makes csv_escape quote it
        put_long(b, (r - beta0) / L + 1);
        b.push_back(',');
        put_long(b, (r - beta0) % L + 1);
        b += "]\"";
      } else {
        b += "gamma[";
        put_long(b, r - gam0 + 1);
        b.push_back(']');
      }
      b.push_back(',');
      put17(b, in.rhat[(size_t)r]);
      b.push_back(',');
      const long col = in.row_col[(size_t)r];
      const int st = col >= 0 ? in.ess_status[(size_t)col] : -1;
      if (st == 0)
        put17(b, in.ess[(size_t)col]);
      else
        b += "NA";
      b.push_back(',');
      const bool degenerate = (in.flags[(size_t)r] & 1) != 0;
      b += degenerate ? "degenerate" : (st < 0 ? "not-retained" : kEss[st]);
      b += (in.flags[(size_t)r] & 2) ? ",1\n" : ",0\n";
    });
    if (!f.ok()) return cannot_write(path, err);
  }

  const long ncol = (long)in.col_names.size();
  for (long c = 0; c < C; ++c) {  // samples/chain_<c>.csv
    const std::string path =
        (root / "samples" / ("chain_" + std::to_string(c + 1) + ".csv")).string();
    RowFile f(path);
    if (!f.ok()) return cannot_write(path, err);
    std::string h = "iteration";
    for (const auto& name : in.col_names) {
      h.push_back(',');
      put_csv(h, name.c_str());
    }
    h.push_back('\n');
    f.put(h);
    const double* s = in.samples.data() + (size_t)c * ncol * in.rows;
    f.rows(in.rows, 64, [&](long r, std::string& b) {
      put_long(b, in.sample_iters[(size_t)r]);
      for (long k = 0; k < ncol; ++k) {
        b.push_back(',');
        put17(b, s[(size_t)k * in.rows + r]);
      }
      b.push_back('\n');
    });
    if (!f.ok()) return cannot_write(path, err);
  }

  {  // run_report.json (io.cpp:665-718)
    Json report;
    report.set("version", Json::S(in.version));
    report.set("seed", Json::U(in.seed));
    report.set("chains", Json::I(in.chains));
    report.set("iterations", Json::I(in.iterations));
    report.set("burnin", Json::I(in.burnin));
    report.set("tune_cutoff", Json::I(in.tune_cutoff));
    report.set("thin", Json::I(in.thin));
    report.set("workers", Json::I(in.workers));
    report.set("max_step_out", Json::I(in.max_step_out));
    report.set("save_genes", Json::I(in.save_genes));
    report.set("sampler_mode", Json::S(in.slice_faithful ? "slice-faithful" : "conjugate-direct"));
    report.set("G", Json::U((unsigned long long)G));
    report.set("N", Json::U((unsigned long long)in.N));
    report.set("L", Json::U((unsigned long long)L));
    report.set("wall_seconds", Json::D(in.wall_seconds));
    Json steps;
    for (int s = 0; s < 7; ++s) {
      double total = 0.0;
      for (long c = 0; c < C; ++c) total += in.step_seconds[(size_t)c][(size_t)s];
      steps.set(kStepNames[s], Json::D(total));
    }
    report.set("step_seconds", steps);
    Json per_chain = Json::A();
    unsigned long long clamp_total = 0;
    for (long c = 0; c < C; ++c) {
      Json entry;
      entry.set("chain", Json::I(c + 1));
      entry.set("clamp_events", Json::U(in.clamp_events[(size_t)c]));
      Json cs;
      for (int s = 0; s < 7; ++s) cs.set(kStepNames[s], Json::D(in.step_seconds[(size_t)c][(size_t)s]));
      entry.set("step_seconds", cs);
      per_chain.arr.push_back(entry);
      clamp_total += in.clamp_events[(size_t)c];
    }
    report.set("per_chain", per_chain);
    report.set("clamp_events", Json::U(clamp_total));
    Json saved = Json::A();
    for (long g : in.saved_genes) saved.arr.push_back(Json::U((unsigned long long)g + 1));
    report.set("saved_genes", saved);
    std::string out;
    report.dump(out, 0);
    out.push_back('\n');
    const std::string path = (root / "run_report.json").string();
    RowFile f(path);
    if (!f.ok()) return cannot_write(path, err);
    f.put(out);
    if (!f.ok()) return cannot_write(path, err);
  }
  return CMC_OK;
}

}  // namespace cmc
