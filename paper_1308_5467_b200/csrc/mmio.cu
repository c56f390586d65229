// mmio.cu — Matrix Market coordinate reader (host code), SURVEY §8(f)-4.
//
// Mirrors load_matrix_market (matrix.py:247-304) + SparseSymmetricMatrix.from_coo
// (matrix.py:46-72): real / integer coordinate files, ``symmetric`` (one
// triangle, expanded) or ``general`` (data must be exactly symmetric) headers,
// duplicates summed, the same ValueError messages.  The assembled CSR has both
// triangles, column indices sorted within each row and duplicates summed in
// file order (the order SciPy's COO -> CSR conversion sees them); the caller
// wraps it as a SparseSymmetricMatrix, and the device matrix layer uploads it
// on first use like any other CSR.  No CUDA calls: it runs without a GPU.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"

struct sdb_mm {
  int64_t n = 0;
  int symmetric_storage = 0;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
  std::vector<double> values;
};

namespace {

std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
    size_t j = i;
    while (j < s.size() && !std::isspace((unsigned char)s[j])) ++j;
    if (j > i) out.emplace_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && std::isspace((unsigned char)s[a])) ++a;
  while (b > a && std::isspace((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

// Python int(): optional sign, digits, surrounding whitespace already split off.
bool parse_int(const std::string& t, int64_t* v) {
  if (t.empty()) return false;
  size_t i = (t[0] == '+' || t[0] == '-') ? 1 : 0;
  if (i == t.size()) return false;
  for (size_t k = i; k < t.size(); ++k)
    if (!std::isdigit((unsigned char)t[k]) && t[k] != '_') return false;
  std::string d;
  for (char c : t)
    if (c != '_') d.push_back(c);
  errno = 0;
  char* end = nullptr;
  long long x = std::strtoll(d.c_str(), &end, 10);
  if (errno || *end) return false;
  *v = x;
  return true;
}

// Python float(): strtod accepts the same decimal / exponent / inf / nan forms
// (correctly rounded on glibc); reject trailing garbage and hex floats.
bool parse_double(const std::string& t, double* v) {
  if (t.empty()) return false;
  for (char c : t)
    if (c == 'x' || c == 'X') return false;
  errno = 0;
  char* end = nullptr;
  double x = std::strtod(t.c_str(), &end);
  if (*end) return false;
  *v = x;
  return true;
}

bool getline_file(FILE* f, std::string* line) {
  line->clear();
  int c;
  bool any = false;
  while ((c = std::fgetc(f)) != EOF) {
    any = true;
    line->push_back((char)c);
    if (c == '\n') break;
  }
  return any;
}

}  // namespace

using namespace sdb;

extern "C" {

int sdb_mm_read(const char* path, sdb_mm** out) {
  SDB_REQUIRE(path && out, "NULL argument");
  *out = nullptr;
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(SDB_EINVAL, "cannot open %s", path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  std::string line;
  getline_file(f, &line);
  auto header = split_ws(line);
  if (header.size() < 5 || header[0] != "%%MatrixMarket")
    return fail(SDB_EINVAL, "not a Matrix Market file (missing %%%%MatrixMarket header)");
  const std::string obj = lower(header[1]), fmt = lower(header[2]), field = lower(header[3]),
                    symmetry = lower(header[4]);
  if (obj != "matrix") return fail(SDB_EINVAL, "unsupported Matrix Market object: %s", obj.c_str());
  if (fmt != "coordinate") return fail(SDB_EINVAL, "unsupported Matrix Market format: %s", fmt.c_str());
  if (field == "complex") return fail(SDB_EINVAL, "complex matrices are not supported");
  if (field != "real" && field != "integer")
    return fail(SDB_EINVAL, "unsupported Matrix Market field: %s", field.c_str());
  if (symmetry != "symmetric" && symmetry != "general")
    return fail(SDB_EINVAL, "unsupported Matrix Market symmetry: %s", symmetry.c_str());

  bool have = getline_file(f, &line);
  while (have && (strip(line).empty() || strip(line)[0] == '%')) have = getline_file(f, &line);
  auto size = split_ws(line);
  if (size.size() != 3) return fail(SDB_EINVAL, "malformed Matrix Market size line");
  int64_t m = 0, n = 0, nnz = 0;
  if (!parse_int(size[0], &m) || !parse_int(size[1], &n) || !parse_int(size[2], &nnz))
    return fail(SDB_EINVAL, "malformed Matrix Market size line");
  if (m != n) return fail(SDB_EINVAL, "matrix must be square, got %lld x %lld", (long long)m, (long long)n);
  if (n < 1 || nnz < 0) return fail(SDB_EINVAL, "invalid Matrix Market dimensions");
  SDB_REQUIRE(n < (1LL << 31), "matrix dimension %lld too large for int32 indices", (long long)n);

  std::vector<int64_t> rows, cols;
  std::vector<double> vals;
  rows.reserve((size_t)nnz);
  cols.reserve((size_t)nnz);
  vals.reserve((size_t)nnz);
  int64_t k = 0;
  while (getline_file(f, &line)) {
    const std::string s = strip(line);
    if (s.empty() || s[0] == '%') continue;
    auto parts = split_ws(s);
    if (parts.size() != 3) return fail(SDB_EINVAL, "malformed coordinate entry: '%s'", s.c_str());
    if (k >= nnz) return fail(SDB_EINVAL, "more entries than declared in size line");
    int64_t i = 0, j = 0;
    double v = 0.0;
    if (!parse_int(parts[0], &i) || !parse_int(parts[1], &j) || !parse_double(parts[2], &v))
      return fail(SDB_EINVAL, "malformed coordinate entry: '%s'", s.c_str());
    if (!(1 <= i && i <= n && 1 <= j && j <= n))
      return fail(SDB_EINVAL, "coordinate index out of range: (%lld, %lld)", (long long)i, (long long)j);
    rows.push_back(i - 1);
    cols.push_back(j - 1);
    vals.push_back(v);
    ++k;
  }
  if (k != nnz) return fail(SDB_EINVAL, "expected %lld entries, found %lld", (long long)nnz, (long long)k);

  // from_coo (matrix.py:46-72): mirrored off-diagonal entries appended after the file's
  const bool sym = symmetry == "symmetric";
  if (sym) {
    const size_t base = rows.size();
    for (size_t e = 0; e < base; ++e)
      if (rows[e] != cols[e]) {
        rows.push_back(cols[e]);
        cols.push_back(rows[e]);
        vals.push_back(vals[e]);
      }
  }
  // COO -> CSR: entries bucketed by row in input order, columns sorted
  // stably within a row, duplicates summed in that order
  const size_t ne = rows.size();
  std::vector<int64_t> count((size_t)n + 1, 0);
  for (size_t e = 0; e < ne; ++e) ++count[(size_t)rows[e] + 1];
  for (int64_t r = 0; r < n; ++r) count[(size_t)r + 1] += count[(size_t)r];
  std::vector<size_t> order(ne);
  {
    std::vector<int64_t> fill(count.begin(), count.end() - 1);
    for (size_t e = 0; e < ne; ++e) order[(size_t)fill[(size_t)rows[e]]++] = e;
  }
  auto* mm = new sdb_mm();
  mm->n = n;
  mm->symmetric_storage = sym ? 1 : 0;
  mm->indptr.assign((size_t)n + 1, 0);
  mm->indices.reserve(ne);
  mm->values.reserve(ne);
  for (int64_t r = 0; r < n; ++r) {
    auto b = order.begin() + count[(size_t)r], en = order.begin() + count[(size_t)r + 1];
    std::stable_sort(b, en, [&](size_t a, size_t c) { return cols[a] < cols[c]; });
    for (auto it = b; it != en; ++it) {
      const int32_t cidx = (int32_t)cols[*it];
      if (!mm->indices.empty() && (int64_t)mm->indices.size() > mm->indptr[(size_t)r] && mm->indices.back() == cidx)
        mm->values.back() += vals[*it];
      else {
        mm->indices.push_back(cidx);
        mm->values.push_back(vals[*it]);
      }
    }
    mm->indptr[(size_t)r + 1] = (int64_t)mm->indices.size();
  }
  // exact symmetry (SparseSymmetricMatrix.is_symmetric, matrix.py:107-109):
  // every stored (i, j, v) has a stored (j, i, v) -- compare with the transpose
  {
    const int64_t nz = (int64_t)mm->indices.size();
    std::vector<int64_t> tptr((size_t)n + 1, 0);
    for (int64_t e = 0; e < nz; ++e) ++tptr[(size_t)mm->indices[(size_t)e] + 1];
    for (int64_t r = 0; r < n; ++r) tptr[(size_t)r + 1] += tptr[(size_t)r];
    std::vector<int32_t> tidx((size_t)nz);
    std::vector<double> tval((size_t)nz);
    std::vector<int64_t> fill(tptr.begin(), tptr.end() - 1);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t e = mm->indptr[(size_t)r]; e < mm->indptr[(size_t)r + 1]; ++e) {
        const int64_t dst = fill[(size_t)mm->indices[(size_t)e]]++;
        tidx[(size_t)dst] = (int32_t)r;
        tval[(size_t)dst] = mm->values[(size_t)e];
      }
    bool same = tptr == mm->indptr && tidx == mm->indices;
    for (int64_t e = 0; same && e < nz; ++e)
      same = tval[(size_t)e] == mm->values[(size_t)e];  // NaN != NaN: not symmetric, as in SciPy
    if (!same) {
      delete mm;
      // load_matrix_market re-raises from_coo's "not symmetric" error with this message
      return fail(SDB_EINVAL, "file declares general symmetry but its data is not symmetric");
    }
  }
  *out = mm;
  return SDB_OK;
}

int sdb_mm_info(const sdb_mm* mm, int64_t* n, int64_t* nnz, int32_t* symmetric_storage) {
  SDB_REQUIRE(mm, "NULL argument");
  if (n) *n = mm->n;
  if (nnz) *nnz = (int64_t)mm->indices.size();
  if (symmetric_storage) *symmetric_storage = mm->symmetric_storage;
  return SDB_OK;
}

int sdb_mm_export(const sdb_mm* mm, int64_t* indptr, int32_t* indices, double* values) {
  SDB_REQUIRE(mm && indptr && (mm->indices.empty() || (indices && values)), "NULL argument");
  std::copy(mm->indptr.begin(), mm->indptr.end(), indptr);
  std::copy(mm->indices.begin(), mm->indices.end(), indices);
  std::copy(mm->values.begin(), mm->values.end(), values);
  return SDB_OK;
}

void sdb_mm_free(sdb_mm* mm) { delete mm; }

}  // extern "C"
