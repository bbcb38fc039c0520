// mm.cu — Matrix Market ingest and output (reference matrix_market.cpp).
//
// Same file semantics as the reference reader/writer (banner checks, comment and blank lines,
// symmetric expansion, pattern option, 1-based line numbers in every parse error, the
// duplicate-summing CSR assembly of sparse.cpp:153-181), built for multi-GB inputs:
//   * the data lines are parsed by all host cores (chunks split at line ends; the first error
//     in file order is the one reported; lines past the declared entry count are ignored, as
//     the reference never reads them);
//   * the triplets are assembled into CSR on the GPU: a stable radix sort by (row, column) and
//     an in-order segment sum (0.0 + v + v' ..., the reference's order), so duplicates and the
//     sign of zero come out exactly as in triplets_to_csr;
//   * the writer formats rows in parallel with the reference's 17-significant-digit to_chars
//     format, so the output is byte-identical and every double round-trips.
#include <cub/cub.cuh>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>

#include "mm.cuh"
#include "primitives.cuh"

namespace aggmg_b200 {

namespace {

[[noreturn]] void fail(int64_t line, const std::string& msg) {
  throw Error("matrix market: line " + std::to_string(line) + ": " + msg);
}

std::string lower(std::string s) {
  for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

struct Banner {
  bool coordinate = false, pattern = false, integer = false, symmetric = false;
};

Banner parse_banner(const std::string& text) {
  std::istringstream f(text);
  std::string tag, object, format, field, symmetry;
  f >> tag >> object >> format >> field >> symmetry;
  if (tag != "%%MatrixMarket") fail(1, "missing %%MatrixMarket banner");
  if (lower(object) != "matrix") fail(1, "unsupported object '" + object + "'");
  Banner b;
  const std::string fmt = lower(format), fld = lower(field), sym = lower(symmetry);
  if (fmt == "coordinate")
    b.coordinate = true;
  else if (fmt != "array")
    fail(1, "unsupported format '" + format + "'");
  if (fld == "pattern")
    b.pattern = true;
  else if (fld == "integer")
    b.integer = true;
  else if (fld != "real")
    fail(1, "unsupported field '" + field + "'");
  if (sym == "symmetric")
    b.symmetric = true;
  else if (sym != "general")
    fail(1, "unsupported symmetry '" + symmetry + "'");
  if (!b.coordinate && b.pattern) fail(1, "array format cannot be pattern");
  return b;
}

// A cursor over one line: the istream >> semantics the reference relies on (skip blanks,
// integers stop at the first non-digit, doubles take the longest numeric prefix).
struct Fields {
  const char* p;
  const char* e;
  void skip() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
  }
  bool integer(long long& v) {
    skip();
    const char* q = p;
    bool neg = false;
    if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
    const auto r = std::from_chars(q, e, v);
    if (r.ec != std::errc() || r.ptr == q) return false;
    if (neg) v = -v;
    p = r.ptr;
    return true;
  }
  bool real(double& v) {
    skip();
    const char* q = p;
    if (q < e && *q == '+') ++q;  // istream accepts a leading plus, from_chars does not
    const auto r = std::from_chars(q, e, v, std::chars_format::general);
    if (r.ec != std::errc() || r.ptr == q) return false;
    p = r.ptr;
    return true;
  }
};

bool content_line(const char* b, const char* e) {
  while (b < e && std::isspace(static_cast<unsigned char>(*b))) ++b;
  return b < e && *b != '%';
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0;    // physical lines in the chunk
  int64_t content = 0;  // content lines (entries)
  int64_t err_content = -1, err_line = -1;  // first failing entry (content index, local line)
  std::string err_msg;
  std::vector<int64_t> ti, tj;
  std::vector<double> tv;
};

void parse_chunk(Chunk& c, const Banner& bn, int64_t n_rows, int64_t n_cols, int64_t limit_hint) {
  const char* p = c.b;
  while (p < c.e) {
    const char* q = static_cast<const char*>(std::memchr(p, '\n', c.e - p));
    const char* le = q ? q : c.e;
    ++c.lines;
    if (content_line(p, le)) {
      const int64_t ci = c.content++;
      if (c.err_content < 0 && ci < limit_hint) {
        Fields f{p, le};
        long long i = 0, j = 0;
        double v = 1.0;
        std::string msg;
        if (!f.integer(i))
          msg = "expected row index";
        else if (!f.integer(j))
          msg = "expected column index";
        else if (!bn.pattern && !f.real(v))
          msg = "expected numeric value";
        else if (i - 1 < 0 || i - 1 >= n_rows || j - 1 < 0 || j - 1 >= n_cols)
          msg = "index out of range";
        else if (bn.symmetric && j > i)
          msg = "symmetric entry above the diagonal";
        if (!msg.empty()) {
          c.err_content = ci;
          c.err_line = c.lines;
          c.err_msg = msg;
        } else {
          c.ti.push_back(i - 1);
          c.tj.push_back(j - 1);
          c.tv.push_back(v);
          if (bn.symmetric && i != j) {
            c.ti.push_back(j - 1);
            c.tj.push_back(i - 1);
            c.tv.push_back(v);
          }
        }
      }
    }
    p = q ? q + 1 : c.e;
  }
}

__global__ void k_keys(const int64_t* ti, const int64_t* tj, int64_t m, int64_t n_cols,
                       unsigned long long* key, int* perm) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  key[k] = static_cast<unsigned long long>(ti[k]) * static_cast<unsigned long long>(n_cols) +
           static_cast<unsigned long long>(tj[k]);
  perm[k] = static_cast<int>(k);
}
// one thread per unique (row, col): the reference's `sum = 0.0; sum += v` in triplet order
__global__ void k_seg_sum(const int* seg_off, int64_t nseg, const int* perm, const double* tv,
                          const unsigned long long* ukey, int64_t n_cols, int64_t* col, double* val,
                          int* row_cnt) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  double sum = 0.0;
  for (int p = seg_off[s]; p < seg_off[s + 1]; ++p) sum = __dadd_rn(sum, tv[perm[p]]);
  val[s] = sum;
  col[s] = static_cast<int64_t>(ukey[s] % static_cast<unsigned long long>(n_cols));
  atomicAdd(&row_cnt[ukey[s] / static_cast<unsigned long long>(n_cols)], 1);
}

template <class F>
void cub_call(F&& f) {
  size_t bytes = 0;
  AGG_CUDA(f(nullptr, bytes));
  DevBuf<char> tmp(static_cast<int64_t>(std::max<size_t>(bytes, 1)));
  AGG_CUDA(f(tmp.get(), bytes));
}

}  // namespace

// triplets_to_csr (sparse.cpp:153-181) on the device
HostCsr triplets_to_csr_device(int64_t n_rows, int64_t n_cols, const std::vector<int64_t>& ti,
                               const std::vector<int64_t>& tj, const std::vector<double>& tv) {
  const int64_t m = static_cast<int64_t>(ti.size());
  require(m < (int64_t{1} << 31), "matrix market: more than 2^31 stored entries");
  HostCsr out;
  out.n = n_rows;
  out.ncols = n_cols;
  out.rp.assign(n_rows + 1, 0);
  if (m == 0) return out;
  DevBuf<int64_t> di(m), dj(m);
  DevBuf<double> dv(m);
  di.upload(ti.data(), m);
  dj.upload(tj.data(), m);
  dv.upload(tv.data(), m);
  DevBuf<unsigned long long> key(m), key_s(m), ukey(m);
  DevBuf<int> perm(m), perm_s(m), seg_len(m), seg_off(m + 1), nseg_d(1);
  AGG_LAUNCH(k_keys, grid_for(m, 256), 256, 0, di.get(), dj.get(), m, n_cols, key.get(), perm.get());
  cub_call([&](void* t, size_t& b) {  // stable: equal (row, col) keep the triplet order
    return cub::DeviceRadixSort::SortPairs(t, b, key.get(), key_s.get(), perm.get(), perm_s.get(),
                                           static_cast<int>(m), 0, 64, stream());
  });
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRunLengthEncode::Encode(t, b, key_s.get(), ukey.get(), seg_len.get(),
                                              nseg_d.get(), static_cast<int>(m), stream());
  });
  const int64_t nseg = read_scalar(nseg_d.get());
  scan_to_offsets_async(seg_len.get(), seg_off.get(), nseg);
  DevBuf<int64_t> col(nseg);
  DevBuf<double> val(nseg);
  DevBuf<int> rcnt(n_rows);
  rcnt.zero();
  AGG_LAUNCH(k_seg_sum, grid_for(nseg, 256), 256, 0, seg_off.get(), nseg, perm_s.get(), dv.get(),
             ukey.get(), n_cols, col.get(), val.get(), rcnt.get());
  out.col.resize(nseg);
  out.val.resize(nseg);
  std::vector<int> rc(n_rows);
  col.download(out.col.data(), nseg);
  val.download(out.val.data(), nseg);
  rcnt.download(rc.data(), n_rows);
  sync();
  for (int64_t i = 0; i < n_rows; ++i) out.rp[i + 1] = out.rp[i] + rc[i];
  return out;
}

HostCsr read_matrix_market_text(const char* data, size_t size, bool allow_pattern) {
  const char* p = data;
  const char* end = data + size;
  const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
  require(size > 0, "matrix market: empty input");
  const Banner bn = parse_banner(std::string(p, nl ? nl : end));
  if (bn.pattern && !allow_pattern) fail(1, "pattern matrices need the pattern option enabled");
  int64_t line = 1;
  p = nl ? nl + 1 : end;
  // size line
  const char* sl = nullptr;
  const char* se = nullptr;
  while (p < end) {
    const char* q = static_cast<const char*>(std::memchr(p, '\n', end - p));
    const char* le = q ? q : end;
    ++line;
    const char* next = q ? q + 1 : end;
    if (content_line(p, le)) {
      sl = p;
      se = le;
      p = next;
      break;
    }
    p = next;
  }
  if (!sl) fail(line + 1, "missing size line");
  Fields sf{sl, se};
  long long n_rows = 0, n_cols = 0, n_stored = 0;
  if (!sf.integer(n_rows)) fail(line, "expected row count");
  if (!sf.integer(n_cols)) fail(line, "expected column count");
  if (bn.coordinate) {
    if (!sf.integer(n_stored)) fail(line, "expected entry count");
    if (n_rows < 0 || n_cols < 0 || n_stored < 0) fail(line, "negative size");
    // parallel parse of the data lines, chunks cut at line ends
    const int nt = static_cast<int>(std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
    const size_t rest = static_cast<size_t>(end - p);
    const int nchunks = rest > (size_t{1} << 22) ? nt : 1;
    std::vector<Chunk> ch(nchunks);
    const char* cb = p;
    for (int c = 0; c < nchunks; ++c) {
      const char* ce = c + 1 == nchunks ? end : std::min(end, p + rest * (c + 1) / nchunks);
      if (ce < end && ce > cb) {
        const char* q = static_cast<const char*>(std::memchr(ce, '\n', end - ce));
        ce = q ? q + 1 : end;
      }
      if (ce < cb) ce = cb;
      ch[c].b = cb;
      ch[c].e = ce;
      cb = ce;
    }
    {
      std::vector<std::thread> th;
      for (int c = 0; c < nchunks; ++c)
        th.emplace_back([&, c] { parse_chunk(ch[c], bn, n_rows, n_cols, INT64_MAX); });
      for (auto& t : th) t.join();
    }
    // first failure within the first n_stored entries, in file order
    int64_t content_before = 0, lines_before = line;
    std::vector<int64_t> ti, tj;
    std::vector<double> tv;
    for (int c = 0; c < nchunks; ++c) {
      Chunk& k = ch[c];
      if (k.err_content >= 0 && content_before + k.err_content < n_stored)
        fail(lines_before + k.err_line, k.err_msg);
      content_before += k.content;
      lines_before += k.lines;
    }
    if (content_before < n_stored) fail(lines_before + 1, "unexpected end of file");
    // keep exactly the first n_stored entries (their triplets, symmetric mirrors included)
    int64_t taken = 0;
    for (int c = 0; c < nchunks && taken < n_stored; ++c) {
      Chunk& k = ch[c];
      if (taken + k.content <= n_stored) {
        ti.insert(ti.end(), k.ti.begin(), k.ti.end());
        tj.insert(tj.end(), k.tj.begin(), k.tj.end());
        tv.insert(tv.end(), k.tv.begin(), k.tv.end());
        taken += k.content;
      } else {  // partial chunk: walk its triplets entry by entry
        size_t t = 0;
        for (int64_t e = 0; e < n_stored - taken; ++e) {
          const bool mirrored = bn.symmetric && k.ti[t] != k.tj[t];
          const size_t cnt = mirrored ? 2 : 1;
          for (size_t u = 0; u < cnt; ++u, ++t) {
            ti.push_back(k.ti[t]);
            tj.push_back(k.tj[t]);
            tv.push_back(k.tv[t]);
          }
        }
        taken = n_stored;
      }
      std::vector<int64_t>().swap(k.ti);
      std::vector<int64_t>().swap(k.tj);
      std::vector<double>().swap(k.tv);
    }
    return triplets_to_csr_device(n_rows, n_cols, ti, tj, tv);
  }
  // array format: dense column-major listing (sequential; dense inputs are small)
  if (n_rows < 0 || n_cols < 0) fail(line, "negative size");
  std::vector<int64_t> ti, tj;
  std::vector<double> tv;
  auto read_entry = [&](int64_t i, int64_t j) {
    const char* ls = nullptr;
    const char* le = nullptr;
    while (p < end) {
      const char* q = static_cast<const char*>(std::memchr(p, '\n', end - p));
      const char* e2 = q ? q : end;
      ++line;
      const char* next = q ? q + 1 : end;
      if (content_line(p, e2)) {
        ls = p;
        le = e2;
        p = next;
        break;
      }
      p = next;
    }
    if (!ls) fail(line + 1, "unexpected end of file");
    Fields f{ls, le};
    double v = 0.0;
    if (!f.real(v)) fail(line, "expected numeric value");
    if (v != 0.0) {
      ti.push_back(i);
      tj.push_back(j);
      tv.push_back(v);
    }
    if (bn.symmetric && i != j && v != 0.0) {
      ti.push_back(j);
      tj.push_back(i);
      tv.push_back(v);
    }
  };
  for (int64_t j = 0; j < n_cols; ++j)
    for (int64_t i = bn.symmetric ? j : 0; i < n_rows; ++i) read_entry(i, j);
  return triplets_to_csr_device(n_rows, n_cols, ti, tj, tv);
}

HostCsr read_matrix_market_file(const std::string& path, bool allow_pattern) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  require(in.good(), "cannot open '" + path + "'");
  const std::streamsize sz = in.tellg();
  in.seekg(0);
  std::string buf(static_cast<size_t>(std::max<std::streamsize>(sz, 0)), '\0');
  if (sz > 0) in.read(&buf[0], sz);
  return read_matrix_market_text(buf.data(), buf.size(), allow_pattern);
}

std::vector<double> read_vector_market_file(const std::string& path) {
  const HostCsr M = read_matrix_market_file(path, false);
  require(M.n > 0 && M.ncols > 0, "matrix market: empty vector");
  require(M.ncols == 1 || M.n == 1, "vector file must have a single column or row, got " +
                                        std::to_string(M.n) + "x" + std::to_string(M.ncols));
  std::vector<double> x(std::max(M.n, M.ncols), 0.0);
  if (M.ncols == 1) {
    for (int64_t i = 0; i < M.n; ++i)
      for (int64_t k = M.rp[i]; k < M.rp[i + 1]; ++k) x[i] = M.val[k];
  } else {
    for (size_t k = 0; k < M.col.size(); ++k) x[M.col[k]] = M.val[k];
  }
  return x;
}

namespace {
inline char* put_double(char* o, double v) {  // 17 significant digits (matrix_market.cpp)
  return std::to_chars(o, o + 32, v, std::chars_format::scientific, 16).ptr;
}
inline char* put_int(char* o, int64_t v) { return std::to_chars(o, o + 24, v).ptr; }
}  // namespace

void write_matrix_market_file(const std::string& path, int64_t n_rows, int64_t n_cols,
                              const int64_t* rp, const int64_t* col, const double* val) {
  std::ofstream out(path, std::ios::binary);
  require(out.good(), "cannot open '" + path + "' for writing");
  const int64_t nnz = rp[n_rows];
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << n_rows << " " << n_cols << " " << nnz << "\n";
  // rows in parallel blocks, each formatted into its own buffer, written in order
  const int nt = static_cast<int>(std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
  const int64_t per_blk = std::max<int64_t>(1, (n_rows + 8 * nt - 1) / (8 * nt));
  const int64_t nblk = (n_rows + per_blk - 1) / per_blk;
  for (int64_t b0 = 0; b0 < nblk; b0 += nt) {
    const int64_t b1 = std::min(nblk, b0 + nt);
    std::vector<std::string> buf(b1 - b0);
    std::vector<std::thread> th;
    for (int64_t b = b0; b < b1; ++b)
      th.emplace_back([&, b] {
        const int64_t r0 = b * per_blk, r1 = std::min(n_rows, r0 + per_blk);
        std::string& s = buf[b - b0];
        s.resize(static_cast<size_t>(rp[r1] - rp[r0]) * 64);
        char* o = &s[0];
        for (int64_t i = r0; i < r1; ++i)
          for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            o = put_int(o, i + 1);
            *o++ = ' ';
            o = put_int(o, col[k] + 1);
            *o++ = ' ';
            o = put_double(o, val[k]);
            *o++ = '\n';
          }
        s.resize(static_cast<size_t>(o - s.data()));
      });
    for (auto& t : th) t.join();
    for (auto& s : buf) out.write(s.data(), static_cast<std::streamsize>(s.size()));
  }
  require(out.good(), "write to '" + path + "' failed");
}

void write_vector_market_file(const std::string& path, const double* x, int64_t n) {
  require(n > 0, "matrix market: empty vector");
  std::ofstream out(path, std::ios::binary);
  require(out.good(), "cannot open '" + path + "' for writing");
  out << "%%MatrixMarket matrix array real general\n";
  out << n << " 1\n";
  std::string s(static_cast<size_t>(n) * 32, '\0');
  char* o = &s[0];
  for (int64_t i = 0; i < n; ++i) {
    o = put_double(o, x[i]);
    *o++ = '\n';
  }
  out.write(s.data(), o - s.data());
  require(out.good(), "write to '" + path + "' failed");
}

}  // namespace aggmg_b200
