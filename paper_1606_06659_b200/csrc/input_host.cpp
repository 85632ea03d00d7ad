// Input side of the path: the count-matrix CSV
// loader and the median-of-ratios offsets, as host C++ in the product
// library.  Both are O(G*N) host work that dominates setup at G = 1M; here
// they run multithreaded.  Results (and error messages) equal the
// reference's load_counts (P:src/io.cpp:125-164, split_csv :46-76,
// parse_count :84-101) and estimate_offsets (P:src/model.cpp:21-68) --
// the offsets bit for bit, since they use the same libm log and the same
// operation order per element.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <string_view>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/countmc_b200.h"

struct cmc_counts {
  long G = 0, N = 0;
  std::unique_ptr<long long[]> counts;  // G x N
  std::string gene_blob, sample_blob;  // NUL-terminated labels, back to back
  std::vector<size_t> gene_off, sample_off;
  bool duplicate_genes = false;
};

struct cmc_table {
  long rows = 0, cols = 0;
  std::vector<double> data;        // rows x cols
  std::vector<std::string> names;  // column names (model matrix: effects)
};

namespace {

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
void parallel_for(long n, long min_chunk, F&& body) {
  const long nt = std::max<long>(1, std::min<long>(n_threads(), n / std::max(1L, min_chunk)));
  if (nt <= 1) {
    body(0L, n, 0);
    return;
  }
  std::vector<std::thread> th;
  const long chunk = (n + nt - 1) / nt;
  for (long t = 0; t < nt; ++t) {
    const long lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([&body, lo, hi, t] { body(lo, hi, (int)t); });
  }
  for (auto& x : th) x.join();
}

// split_csv (P:src/io.cpp:46-76): a quote opens quoting only at the start
// of a cell; "" inside quotes is a literal quote.
void split_csv(const char* b, const char* e, std::vector<std::string>& out) {
  out.clear();
  std::string cur;
  bool quoted = false;
  for (const char* p = b; p < e; ++p) {
    const char ch = *p;
    if (quoted) {
      if (ch == '"') {
        if (p + 1 < e && p[1] == '"') {
          cur += '"';
          ++p;
        } else {
          quoted = false;
        }
      } else {
        cur += ch;
      }
    } else if (ch == '"' && cur.empty()) {
      quoted = true;
    } else if (ch == ',') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += ch;
    }
  }
  out.push_back(cur);
}

// parse_count (P:src/io.cpp:84-101): strtoll base 10 over the whole cell.
// Cells of 1-18 plain digits (no sign, no blanks, cannot overflow) take the
// fast path; everything else goes through strtoll itself.  Returns 0 ok,
// 1 non-integer, 2 negative.
int parse_cell(const char* b, const char* e, long long* v) {
  const long len = e - b;
  if (len >= 1 && len <= 18) {
    long long x = 0;
    const char* p = b;
    for (; p < e; ++p) {
      const unsigned d = (unsigned)(*p - '0');
      if (d > 9) break;
      x = x * 10 + d;
    }
    if (p == e) {
      *v = x;
      return 0;
    }
  }
  std::string cell(b, e);
  errno = 0;
  char* end = nullptr;
  const long long x = std::strtoll(cell.c_str(), &end, 10);
  if (cell.empty() || end != cell.c_str() + cell.size() || errno == ERANGE) return 1;
  *v = x;
  return x < 0 ? 2 : 0;
}

struct RowError {
  long line = -1;  // 0-based line index in the file
  std::string msg;
};

struct ThreadOut {
  std::string blob;
  std::vector<size_t> off;
  RowError err;
};

std::string cell_error(int kind, const std::string& cell, long long v, const std::string& gene,
                       const std::string& sample, long row, long col) {
  std::ostringstream msg;
  if (kind == 1)
    msg << "non-integer count '" << cell << "' for gene '" << gene << "', sample '" << sample
        << "' (row " << row << ", column " << col << ")";
  else
    msg << "negative count " << v << " for gene '" << gene << "', sample '" << sample
        << "' (row " << row << ", column " << col << ")";
  return msg.str();
}

// Parses one data row into counts[0..N) and appends its gene label to out.
// Returns false (with out.err set) on the reference's first error.
bool parse_row(const char* b, const char* e, long N, long row, long li,
               const std::vector<std::string>& samples, long long* counts, ThreadOut& out,
               std::vector<std::string>& parts) {
  if (std::memchr(b, '"', (size_t)(e - b)) == nullptr) {
    // quote-free: cells are exactly the comma-separated spans
    const char* p = b;
    const char* gend = static_cast<const char*>(std::memchr(p, ',', (size_t)(e - p)));
    long n = 0;
    bool ok = gend != nullptr;
    if (ok) {
      p = gend + 1;
      for (; n < N; ++n) {
        const char* c = static_cast<const char*>(std::memchr(p, ',', (size_t)(e - p)));
        const char* ce = c ? c : e;
        if (!c && n != N - 1) break;      // too few cells
        if (c && n == N - 1) break;       // too many cells
        long long v = 0;
        const int kind = parse_cell(p, ce, &v);
        if (kind) {
          const std::string gene(b, gend);
          out.err = {li, cell_error(kind, std::string(p, ce), v, gene, samples[n], row, n + 2)};
          return false;
        }
        counts[n] = v;
        p = ce + 1;
      }
    }
    if (ok && n == N) {
      out.off.push_back(out.blob.size());
      out.blob.append(b, gend);
      out.blob.push_back('\0');
      return true;
    }
    // wrong cell count: fall through to the general path for the message
  }
  split_csv(b, e, parts);
  if ((long)parts.size() != N + 1) {
    std::ostringstream msg;
    msg << "row " << row << " has " << parts.size() << " cells, expected " << (N + 1);
    out.err = {li, msg.str()};
    return false;
  }
  for (long n = 0; n < N; ++n) {
    const std::string& cell = parts[n + 1];
    long long v = 0;
    const int kind = parse_cell(cell.data(), cell.data() + cell.size(), &v);
    if (kind) {
      out.err = {li, cell_error(kind, cell, v, parts[0], samples[n], row, n + 2)};
      return false;
    }
    counts[n] = v;
  }
  out.off.push_back(out.blob.size());
  out.blob.append(parts[0]);
  out.blob.push_back('\0');
  return true;
}

long strip_cr(const char* buf, long s, long e) { return (e > s && buf[e - 1] == '\r') ? e - 1 : e; }

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

// The whole file, mapped read-only when it is a regular file (page-ins then
// happen inside the parallel passes), else read through stdio.
struct FileBytes {
  const char* data = nullptr;
  long size = 0;
  void* map = nullptr;
  std::string copy;
  bool open(const char* path) {
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return false;
    struct stat st;
    if (fstat(fd, &st) == 0 && S_ISREG(st.st_mode) && st.st_size > 0) {
      void* p = mmap(nullptr, (size_t)st.st_size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (p != MAP_FAILED) {
        map = p;
        data = static_cast<const char*>(p);
        size = (long)st.st_size;
        ::close(fd);
        return true;
      }
    }
    char chunk[1 << 16];
    ssize_t r;
    while ((r = ::read(fd, chunk, sizeof(chunk))) > 0) copy.append(chunk, (size_t)r);
    ::close(fd);
    if (r < 0) return false;
    data = copy.data();
    size = (long)copy.size();
    return true;
  }
  ~FileBytes() {
    if (map) munmap(map, (size_t)size);
  }
};

// duplicate_genes (io.cpp:151): any label seen twice.  Rows are sharded by
// hash over T threads, each probing its own open-addressing table.
bool any_duplicate(const cmc_counts& m, const std::vector<uint64_t>& hashes, int T) {
  const long G = m.G;
  std::vector<char> dup((size_t)T, 0);
  run_threads(T, [&](int t) {
    size_t cap = 16;
    while (cap < 2 * (size_t)(G / T + 1)) cap <<= 1;
    std::vector<long> table(cap, -1);
    for (long g = 0; g < G; ++g) {
      const uint64_t h = hashes[(size_t)g];
      if ((long)((h >> 40) % (uint64_t)T) != t) continue;
      const char* label = m.gene_blob.data() + m.gene_off[(size_t)g];
      for (size_t i = h & (cap - 1);; i = (i + 1) & (cap - 1)) {
        const long o = table[i];
        if (o < 0) {
          table[i] = g;
          break;
        }
        if (hashes[(size_t)o] == h && std::strcmp(m.gene_blob.data() + m.gene_off[(size_t)o], label) == 0) {
          dup[(size_t)t] = 1;
          return;
        }
      }
    }
  });
  for (char d : dup)
    if (d) return true;
  return false;
}

}  // namespace

extern "C" {

int cmc_counts_load(const char* path, cmc_counts** out, cmc_error* err) {
  if (!path || !out) {
    set_err(err, CMC_ERR_ARG, "null argument");
    return CMC_ERR_ARG;
  }
  *out = nullptr;
  FileBytes file;
  if (!file.open(path)) {
    set_err(err, CMC_ERR_LOAD, std::string("cannot open counts file '") + path + "'");
    return CMC_ERR_LOAD;
  }
  const char* buf = file.data;
  const long nbytes = file.size;
  if (nbytes == 0) {
    set_err(err, CMC_ERR_LOAD, std::string("counts file '") + path + "' is empty");
    return CMC_ERR_LOAD;
  }
  // header = first line (read_line: getline on '\n', strip one '\r')
  const char* nl0 = static_cast<const char*>(std::memchr(buf, '\n', (size_t)nbytes));
  const long h_end = nl0 ? (long)(nl0 - buf) : nbytes;
  std::vector<std::string> header;
  split_csv(buf, buf + strip_cr(buf, 0, h_end), header);
  if (header.size() < 2) {
    set_err(err, CMC_ERR_LOAD, "counts header needs a gene column plus sample columns");
    return CMC_ERR_LOAD;
  }
  auto m = std::make_unique<cmc_counts>();
  const std::vector<std::string> samples(header.begin() + 1, header.end());
  const long N = (long)samples.size();

  // body split into newline-aligned chunks, one per thread
  const long body = nl0 ? h_end + 1 : nbytes;
  const int T = (int)std::max<long>(1, std::min<long>(n_threads(), (nbytes - body) / (1 << 16)));
  std::vector<long> cut((size_t)T + 1, nbytes);
  cut[0] = body;
  for (int t = 1; t < T; ++t) {
    long c = body + (nbytes - body) * t / T;
    c = std::max(c, cut[(size_t)t - 1]);
    const void* nl = c < nbytes ? std::memchr(buf + c, '\n', (size_t)(nbytes - c)) : nullptr;
    cut[(size_t)t] = nl ? (long)((const char*)nl - buf) + 1 : nbytes;
  }
  // pass 1: lines and non-empty (data) lines per chunk
  std::vector<long> n_lines((size_t)T), n_rows((size_t)T);
  run_threads(T, [&](int t) {
    long lines = 0, rows = 0;
    for (long s = cut[(size_t)t]; s < cut[(size_t)t + 1];) {
      const void* nl = std::memchr(buf + s, '\n', (size_t)(cut[(size_t)t + 1] - s));
      const long e = nl ? (long)((const char*)nl - buf) : cut[(size_t)t + 1];
      ++lines;
      rows += strip_cr(buf, s, e) > s;
      s = e + 1;
    }
    n_lines[(size_t)t] = lines;
    n_rows[(size_t)t] = rows;
  });
  std::vector<long> line0((size_t)T), row0((size_t)T);
  long G = 0, L = 1;
  for (int t = 0; t < T; ++t) {
    line0[(size_t)t] = L;
    row0[(size_t)t] = G;
    L += n_lines[(size_t)t];
    G += n_rows[(size_t)t];
  }
  if (G == 0) {
    set_err(err, CMC_ERR_LOAD, "counts file has no gene rows");
    return CMC_ERR_LOAD;
  }
  m->G = G;
  m->N = N;
  m->counts.reset(new long long[(size_t)G * N]);  // first touched by the parsing threads
  std::vector<uint64_t> hashes((size_t)G);
  // pass 2: parse rows in place
  std::vector<ThreadOut> outs((size_t)T);
  run_threads(T, [&](int t) {
    ThreadOut& o = outs[(size_t)t];
    o.off.reserve((size_t)n_rows[(size_t)t]);
    std::vector<std::string> parts;
    long li = line0[(size_t)t], r = row0[(size_t)t];
    for (long s = cut[(size_t)t]; s < cut[(size_t)t + 1]; ++li) {
      const void* nl = std::memchr(buf + s, '\n', (size_t)(cut[(size_t)t + 1] - s));
      const long e = nl ? (long)((const char*)nl - buf) : cut[(size_t)t + 1];
      const long ee = strip_cr(buf, s, e);
      if (ee > s) {
        // li is the 0-based file line, so the reference's 1-based row is li + 1
        if (!parse_row(buf + s, buf + ee, N, li + 1, li, samples, &m->counts[(size_t)r * N], o,
                       parts))
          return;
        const size_t k = o.off.back();
        hashes[(size_t)r] = std::hash<std::string_view>()(
            std::string_view(o.blob.data() + k, o.blob.size() - 1 - k));
        ++r;
      }
      s = e + 1;
    }
  });
  // the reference stops at the first bad row in file order
  const RowError* first = nullptr;
  for (const auto& o : outs)
    if (o.err.line >= 0 && (!first || o.err.line < first->line)) first = &o.err;
  if (first) {
    set_err(err, CMC_ERR_LOAD, first->msg);
    return CMC_ERR_LOAD;
  }
  size_t total = 0;
  for (const auto& o : outs) total += o.blob.size();
  m->gene_blob.resize(total);
  m->gene_off.resize((size_t)G);
  {
    std::vector<size_t> base((size_t)T);
    size_t acc = 0;
    for (int t = 0; t < T; ++t) {
      base[(size_t)t] = acc;
      acc += outs[(size_t)t].blob.size();
    }
    run_threads(T, [&](int t) {
      const ThreadOut& o = outs[(size_t)t];
      std::memcpy(&m->gene_blob[base[(size_t)t]], o.blob.data(), o.blob.size());
      for (size_t k = 0; k < o.off.size(); ++k)
        m->gene_off[(size_t)row0[(size_t)t] + k] = base[(size_t)t] + o.off[k];
    });
  }
  for (const auto& s : samples) {
    m->sample_off.push_back(m->sample_blob.size());
    m->sample_blob.append(s);
    m->sample_blob.push_back('\0');
  }
  m->duplicate_genes = any_duplicate(*m, hashes, T);
  *out = m.release();
  return CMC_OK;
}

int cmc_counts_dims(const cmc_counts* c, long* G, long* N, int* duplicate_genes) {
  if (!c) return CMC_ERR_ARG;
  if (G) *G = c->G;
  if (N) *N = c->N;
  if (duplicate_genes) *duplicate_genes = c->duplicate_genes ? 1 : 0;
  return CMC_OK;
}

const long long* cmc_counts_data(const cmc_counts* c) { return c ? c->counts.get() : nullptr; }

const char* cmc_counts_gene(const cmc_counts* c, long g) {
  return (c && g >= 0 && g < c->G) ? c->gene_blob.data() + c->gene_off[(size_t)g] : nullptr;
}

const char* cmc_counts_sample(const cmc_counts* c, long n) {
  return (c && n >= 0 && n < c->N) ? c->sample_blob.data() + c->sample_off[(size_t)n] : nullptr;
}

int cmc_counts_labels(const cmc_counts* c, int which, const char** blob, size_t* bytes) {
  if (!c || !blob || !bytes || (which != 0 && which != 1)) return CMC_ERR_ARG;
  const std::string& b = which == 0 ? c->gene_blob : c->sample_blob;
  *blob = b.data();
  *bytes = b.size();
  return CMC_OK;
}

void cmc_counts_free(cmc_counts* c) { delete c; }

// ---- the small tables of the input side: read like the reference
// (std::getline, one trailing '\r' stripped, blank rows skipped), cells by
// split_csv, numbers by strtod over the whole cell (parse_real,
// P:src/io.cpp:103-114, errno not consulted).
namespace {

bool read_line(std::ifstream& in, std::string& line) {
  if (!std::getline(in, line)) return false;
  if (!line.empty() && line.back() == '\r') line.pop_back();
  return true;
}

bool parse_real(const std::string& cell, double* v) {
  char* end = nullptr;
  *v = std::strtod(cell.c_str(), &end);
  return !cell.empty() && end == cell.c_str() + cell.size();
}

std::string malformed(const char* what, const std::string& cell, long row, long col) {
  std::ostringstream msg;
  msg << "malformed " << what << " '" << cell << "' (row " << row << ", column " << col << ")";
  return msg.str();
}

}  // namespace

extern "C" {

// load_model_matrix, P:src/io.cpp:178-205: header = effect names (L cells),
// one row per sample with L numbers.
int cmc_model_matrix_load(const char* path, cmc_table** out, cmc_error* err) {
  if (!path || !out) {
    set_err(err, CMC_ERR_ARG, "null argument");
    return CMC_ERR_ARG;
  }
  *out = nullptr;
  std::ifstream in(path);
  if (!in) {
    set_err(err, CMC_ERR_LOAD, std::string("cannot open model matrix file '") + path + "'");
    return CMC_ERR_LOAD;
  }
  std::string line;
  if (!read_line(in, line)) {
    set_err(err, CMC_ERR_LOAD, std::string("model matrix file '") + path + "' is empty");
    return CMC_ERR_LOAD;
  }
  auto t = std::make_unique<cmc_table>();
  split_csv(line.data(), line.data() + line.size(), t->names);
  const long L = (long)t->names.size();
  std::vector<std::string> parts;
  long row = 1;
  while (read_line(in, line)) {
    ++row;
    if (line.empty()) continue;
    split_csv(line.data(), line.data() + line.size(), parts);
    if ((long)parts.size() != L) {
      std::ostringstream msg;
      msg << "model matrix row " << row << " has " << parts.size() << " cells, expected " << L;
      set_err(err, CMC_ERR_LOAD, msg.str());
      return CMC_ERR_LOAD;
    }
    for (long l = 0; l < L; ++l) {
      double v;
      if (!parse_real(parts[(size_t)l], &v)) {
        set_err(err, CMC_ERR_LOAD, malformed("model matrix entry", parts[(size_t)l], row, l + 1));
        return CMC_ERR_LOAD;
      }
      t->data.push_back(v);
    }
    ++t->rows;
  }
  if (t->rows == 0) {
    set_err(err, CMC_ERR_LOAD, "model matrix has no rows");
    return CMC_ERR_LOAD;
  }
  t->cols = L;
  *out = t.release();
  return CMC_OK;
}

// load_offsets, P:src/io.cpp:221-243: header line, then "sample,offset"
// rows; the offset is the second cell.
int cmc_offsets_load(const char* path, cmc_table** out, cmc_error* err) {
  if (!path || !out) {
    set_err(err, CMC_ERR_ARG, "null argument");
    return CMC_ERR_ARG;
  }
  *out = nullptr;
  std::ifstream in(path);
  if (!in) {
    set_err(err, CMC_ERR_LOAD, std::string("cannot open offsets file '") + path + "'");
    return CMC_ERR_LOAD;
  }
  std::string line;
  if (!read_line(in, line)) {
    set_err(err, CMC_ERR_LOAD, std::string("offsets file '") + path + "' is empty");
    return CMC_ERR_LOAD;
  }
  auto t = std::make_unique<cmc_table>();
  t->names = {"offset"};
  std::vector<std::string> parts;
  long row = 1;
  while (read_line(in, line)) {
    ++row;
    if (line.empty()) continue;
    split_csv(line.data(), line.data() + line.size(), parts);
    if (parts.size() != 2) {
      std::ostringstream msg;
      msg << "offsets row " << row << " has " << parts.size() << " cells, expected 2";
      set_err(err, CMC_ERR_LOAD, msg.str());
      return CMC_ERR_LOAD;
    }
    double v;
    if (!parse_real(parts[1], &v)) {
      set_err(err, CMC_ERR_LOAD, malformed("offset", parts[1], row, 2));
      return CMC_ERR_LOAD;
    }
    t->data.push_back(v);
    ++t->rows;
  }
  if (t->rows == 0) {
    set_err(err, CMC_ERR_LOAD, "offsets file has no rows");
    return CMC_ERR_LOAD;
  }
  t->cols = 1;
  *out = t.release();
  return CMC_OK;
}

int cmc_table_dims(const cmc_table* t, long* rows, long* cols) {
  if (!t) return CMC_ERR_ARG;
  if (rows) *rows = t->rows;
  if (cols) *cols = t->cols;
  return CMC_OK;
}

const double* cmc_table_data(const cmc_table* t) { return t ? t->data.data() : nullptr; }

const char* cmc_table_name(const cmc_table* t, long col) {
  return (t && col >= 0 && col < (long)t->names.size()) ? t->names[(size_t)col].c_str() : nullptr;
}

void cmc_table_free(cmc_table* t) { delete t; }

}  // extern "C"

// estimate_offsets, P:src/model.cpp:21-68: log geometric mean per gene over
// genes positive in every sample, per-sample median of log ratios
// (std::sort, midpoint average for even counts), recentred to sum zero.
int cmc_estimate_offsets(long G, long N, const long long* counts, double* h,
                         cmc_error* err) {
  if (G < 1 || N < 1 || !counts || !h) {
    set_err(err, CMC_ERR_ARG, "bad arguments");
    return CMC_ERR_ARG;
  }
  // log(y) for small counts memoised: glibc log is a pure function of its
  // argument, so the table holds exactly the values the reference computes
  constexpr long kLogTab = 1 << 16;
  std::vector<double> logtab(kLogTab);
  parallel_for(kLogTab, 8192, [&](long lo, long hi, int) {
    for (long k = lo; k < hi; ++k) logtab[(size_t)k] = std::log(static_cast<double>(k));
  });
  auto logy = [&](long long y) {
    return y < kLogTab ? logtab[(size_t)y] : std::log(static_cast<double>(y));
  };
  std::vector<double> loggm_all((size_t)G);
  std::vector<char> pos((size_t)G);
  parallel_for(G, 8192, [&](long lo, long hi, int) {
    for (long g = lo; g < hi; ++g) {
      bool positive = true;
      double slog = 0.0;
      for (long n = 0; n < N; ++n) {
        const long long y = counts[(size_t)g * N + n];
        if (y <= 0) {
          positive = false;
          break;
        }
        slog += logy(y);
      }
      pos[(size_t)g] = positive;
      loggm_all[(size_t)g] = slog / static_cast<double>(N);
    }
  });
  std::vector<long> keep;
  std::vector<double> loggm;
  for (long g = 0; g < G; ++g)
    if (pos[(size_t)g]) {
      keep.push_back(g);
      loggm.push_back(loggm_all[(size_t)g]);
    }
  if (keep.empty()) {
    set_err(err, CMC_ERR_CONFIG,
            "offset estimation needs at least one gene with positive counts in "
            "every sample; supply offsets explicitly instead");
    return CMC_ERR_CONFIG;
  }
  std::vector<double> med((size_t)N);
  parallel_for(N, 1, [&](long lo, long hi, int) {
    std::vector<double> ratios(keep.size());
    for (long n = lo; n < hi; ++n) {
      for (size_t i = 0; i < keep.size(); ++i)
        ratios[i] = logy(counts[(size_t)keep[i] * N + n]) - loggm[i];
      // the reference sorts; selection yields the same order statistics
      const size_t k = ratios.size();
      std::nth_element(ratios.begin(), ratios.begin() + k / 2, ratios.end());
      const double hi = ratios[k / 2];
      if (k % 2 == 1) {
        med[(size_t)n] = hi;
      } else {
        const double lo = *std::max_element(ratios.begin(), ratios.begin() + k / 2);
        med[(size_t)n] = 0.5 * (lo + hi);
      }
    }
  });
  double mean = 0.0;
  for (long n = 0; n < N; ++n) mean += med[(size_t)n];
  mean /= static_cast<double>(N);
  for (long n = 0; n < N; ++n) h[n] = med[(size_t)n] - mean;
  return CMC_OK;
}

}  // extern "C"
