// bo_io.cpp — MatrixMarket ingestion for the matrix-powers operator (host).
//
// Same grammar, error texts and CSR as the reference's read_matrix_market /
// write_matrix_market (proj/src/sparse.cpp:88-152) and
// CsrMatrix::from_triplets (proj/src/sparse.cpp:13-42): "matrix coordinate
// real general|symmetric", 1-based indices, symmetric entries mirrored,
// entries sorted by (row, col) with std::sort and duplicates summed in that
// order, so the values are bit-identical for the same libstdc++.
#include <algorithm>
#include <cctype>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/bo_cuda.h"

struct bo_csr_host_s {
  uint64_t nrows = 0, ncols = 0;
  std::vector<int64_t> row_ptr, col;
  std::vector<double> val;
};

namespace {
struct Trip {
  uint64_t row, col;
  double value;
};

int fail(bo_status* st, int code, const std::string& msg, long long index = 0) {
  if (st) {
    st->code = code;
    st->index = index;
    st->pivot = 0.0;
    std::snprintf(st->msg, sizeof st->msg, "%s", msg.c_str());
  }
  return code;
}
std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}
int parse_error(bo_status* st, size_t line, const std::string& msg) {  // errors.hpp:77-86
  return fail(st, BO_PARSE_ERROR, "parse error at line " + std::to_string(line) + ": " + msg, (long long)line);
}
int banner_error(bo_status* st, const std::string& banner) {  // errors.hpp:88-92
  return fail(st, BO_BANNER_ERROR, "unsupported MatrixMarket banner: " + banner);
}

// CsrMatrix::from_triplets (sparse.cpp:13-42)
void from_triplets(bo_csr_host_s& m, uint64_t nrows, uint64_t ncols, std::vector<Trip> e) {
  std::sort(e.begin(), e.end(),
            [](const Trip& a, const Trip& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
  m.nrows = nrows;
  m.ncols = ncols;
  m.row_ptr.assign(nrows + 1, 0);
  m.col.reserve(e.size());
  m.val.reserve(e.size());
  for (size_t i = 0; i < e.size();) {
    const uint64_t r = e[i].row, c = e[i].col;
    double v = 0.0;
    while (i < e.size() && e[i].row == r && e[i].col == c) {
      v += e[i].value;
      ++i;
    }
    m.col.push_back((int64_t)c);
    m.val.push_back(v);
    m.row_ptr[r + 1] = (int64_t)m.col.size();
  }
  for (uint64_t r = 0; r < nrows; ++r) m.row_ptr[r + 1] = std::max(m.row_ptr[r + 1], m.row_ptr[r]);
}
}  // namespace

extern "C" int bo_mm_read(const char* path, bo_csr_host* out, bo_status* st) {
  if (st) std::memset(st, 0, sizeof *st);
  *out = nullptr;
  const std::string p = path ? path : "";
  std::ifstream in(p);
  if (!in) return parse_error(st, 0, "cannot open file '" + p + "'");
  std::string line;
  size_t lineno = 0;
  if (!std::getline(in, line)) return parse_error(st, 1, "empty file");
  ++lineno;
  std::istringstream banner(line);
  std::string tag, object, format, field, symmetry;
  banner >> tag >> object >> format >> field >> symmetry;
  if (tag != "%%MatrixMarket") return banner_error(st, line);
  object = lower(object);
  format = lower(format);
  field = lower(field);
  symmetry = lower(symmetry);
  if (object != "matrix" || format != "coordinate" || field != "real" ||
      (symmetry != "general" && symmetry != "symmetric"))
    return banner_error(st, line);
  const bool symmetric = symmetry == "symmetric";
  size_t nrows = 0, ncols = 0, nnz = 0;
  bool have_sizes = false;
  std::vector<Trip> entries;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty() || line[0] == '%') continue;
    std::istringstream ls(line);
    if (!have_sizes) {
      if (!(ls >> nrows >> ncols >> nnz)) return parse_error(st, lineno, "bad size line");
      have_sizes = true;
      entries.reserve(symmetric ? 2 * nnz : nnz);
      continue;
    }
    long long r = 0, c = 0;
    double v = 0.0;
    if (!(ls >> r >> c >> v)) return parse_error(st, lineno, "bad entry line");
    if (r < 1 || c < 1 || (size_t)r > nrows || (size_t)c > ncols) return parse_error(st, lineno, "index out of range");
    const uint64_t ri = (uint64_t)(r - 1), cj = (uint64_t)(c - 1);
    entries.push_back({ri, cj, v});
    if (symmetric && ri != cj) entries.push_back({cj, ri, v});
  }
  if (!have_sizes) return parse_error(st, lineno, "missing size line");
  auto* m = new bo_csr_host_s();
  from_triplets(*m, nrows, ncols, std::move(entries));
  *out = m;
  return BO_OK;
}

extern "C" int bo_csr_host_info(bo_csr_host h, uint64_t* nrows, uint64_t* ncols, uint64_t* nnz) {
  if (!h) return BO_INVALID;
  *nrows = h->nrows;
  *ncols = h->ncols;
  *nnz = h->val.size();
  return BO_OK;
}

extern "C" int bo_csr_host_arrays(bo_csr_host h, int64_t* row_ptr, int64_t* col, double* val) {
  if (!h) return BO_INVALID;
  std::copy(h->row_ptr.begin(), h->row_ptr.end(), row_ptr);
  std::copy(h->col.begin(), h->col.end(), col);
  std::copy(h->val.begin(), h->val.end(), val);
  return BO_OK;
}

extern "C" int bo_csr_host_destroy(bo_csr_host h) {
  delete h;
  return BO_OK;
}

// write_matrix_market (sparse.cpp:138-152): general banner, 17 significant digits
extern "C" int bo_mm_write(const char* path, uint64_t nrows, uint64_t ncols, const int64_t* row_ptr,
                           const int64_t* col, const double* val, bo_status* st) {
  if (st) std::memset(st, 0, sizeof *st);
  const std::string p = path ? path : "";
  std::ofstream out(p);
  if (!out) return parse_error(st, 0, "cannot open file '" + p + "' for writing");
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << nrows << " " << ncols << " " << (uint64_t)(row_ptr[nrows] - row_ptr[0]) << "\n";
  out.precision(17);
  for (uint64_t r = 0; r < nrows; ++r)
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) out << r + 1 << " " << col[k] + 1 << " " << val[k] << "\n";
  return BO_OK;
}
