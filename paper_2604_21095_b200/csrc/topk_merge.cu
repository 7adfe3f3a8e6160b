// Host-side merge step of the TOPK writer (reference output.TopKWriter.emit, output.py:155-213):
// the records held so far (sorted by phenotype, then p, then marker source index) and a batch's
// new candidates are merged per phenotype and the first k of each phenotype kept, in that order.
// A batch's candidates all come from markers later in the source than every held record, so
// the (p, source index) order puts a held record before a new one of equal p — as the
// reference's heaps do. Counting sort of the candidates by phenotype, a sort of each
// phenotype's few candidates, then a k-bounded two-way merge, phenotypes in parallel; the
// Python writer only gathers its columns through the returned indices.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "pg_common.cuh"

extern "C" {

// held_*: n_held records sorted by (col, p, src); fresh_*: n_fresh records in any order.
// out_idx (capacity n_pheno * k): indices into [held ++ fresh] of the kept records, sorted by
// (col, p, src); *n_out their count.
int pg_topk_merge(int64_t n_pheno, int64_t k, const int64_t* held_col, const double* held_p, const int64_t* held_src,
                  int64_t n_held, const int64_t* fresh_col, const double* fresh_p, const int64_t* fresh_src,
                  int64_t n_fresh, int64_t* out_idx, int64_t* n_out) {
  PG_REQUIRE(n_pheno >= 1 && k >= 1 && n_held >= 0 && n_fresh >= 0 && out_idx != nullptr && n_out != nullptr,
             PG_ERR_INVALID, "pg_topk_merge: bad arguments");
  // held segment of each phenotype
  std::vector<int64_t> h_begin(n_pheno + 1, 0);
  for (int64_t i = 0; i < n_held; ++i) {
    const int64_t c = held_col[i];
    PG_REQUIRE(c >= 0 && c < n_pheno, PG_ERR_INVALID, "pg_topk_merge: phenotype index out of range");
    ++h_begin[c + 1];
  }
  for (int64_t c = 0; c < n_pheno; ++c) h_begin[c + 1] += h_begin[c];
  // candidates bucketed by phenotype (counting sort; stable)
  std::vector<int64_t> f_begin(n_pheno + 1, 0);
  for (int64_t i = 0; i < n_fresh; ++i) {
    const int64_t c = fresh_col[i];
    PG_REQUIRE(c >= 0 && c < n_pheno, PG_ERR_INVALID, "pg_topk_merge: phenotype index out of range");
    ++f_begin[c + 1];
  }
  for (int64_t c = 0; c < n_pheno; ++c) f_begin[c + 1] += f_begin[c];
  std::vector<int64_t> f_order(static_cast<size_t>(n_fresh));
  {
    std::vector<int64_t> fill(f_begin.begin(), f_begin.end() - 1);
    for (int64_t i = 0; i < n_fresh; ++i) f_order[fill[fresh_col[i]]++] = i;
  }
  // kept count per phenotype -> output offsets
  std::vector<int64_t> out_begin(n_pheno + 1, 0);
  for (int64_t c = 0; c < n_pheno; ++c)
    out_begin[c + 1] = out_begin[c] + std::min<int64_t>(k, (h_begin[c + 1] - h_begin[c]) + (f_begin[c + 1] - f_begin[c]));
  auto less_fresh = [&](int64_t a, int64_t b) {
    return fresh_p[a] < fresh_p[b] || (fresh_p[a] == fresh_p[b] && fresh_src[a] < fresh_src[b]);
  };
  auto work = [&](int64_t c_lo, int64_t c_hi) {
    for (int64_t c = c_lo; c < c_hi; ++c) {
      int64_t* fb = f_order.data() + f_begin[c];
      int64_t* fe = f_order.data() + f_begin[c + 1];
      const int64_t want = out_begin[c + 1] - out_begin[c];
      if (fe - fb > want) {
        std::partial_sort(fb, fb + want, fe, less_fresh);  // only the best `want` can be kept
        fe = fb + want;
      } else {
        std::sort(fb, fe, less_fresh);
      }
      int64_t h = h_begin[c];
      const int64_t he = h_begin[c + 1];
      int64_t* out = out_idx + out_begin[c];
      for (int64_t j = 0; j < want; ++j) {
        // a held record wins ties: its source index is below every candidate's
        const bool take_held =
            h < he && (fb == fe || held_p[h] < fresh_p[*fb] || (held_p[h] == fresh_p[*fb] && held_src[h] < fresh_src[*fb]));
        out[j] = take_held ? h++ : n_held + *fb++;
      }
    }
  };
  const int64_t total = n_held + n_fresh;
  const int nt = total < (1 << 16) ? 1 : static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  if (nt == 1) {
    work(0, n_pheno);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(work, n_pheno * t / nt, n_pheno * (t + 1) / nt);
    for (auto& x : th) x.join();
  }
  *n_out = out_begin[n_pheno];
  return PG_OK;
}

// out_cols[c][i] = (idx[i] < n_held ? held_cols[c][idx[i]] : fresh_cols[c][idx[i] - n_held]) for the
// n_cols 8-byte columns of the TOPK writer (the merge's gather, on host threads).
int pg_topk_gather(int64_t n_out, const int64_t* idx, int64_t n_held, int n_cols, const void* const* held_cols,
                   const void* const* fresh_cols, void* const* out_cols) {
  PG_REQUIRE(n_out >= 0 && n_cols >= 0 && (n_out == 0 || (idx && held_cols && fresh_cols && out_cols)), PG_ERR_INVALID,
             "pg_topk_gather: bad arguments");
  auto work = [&](int64_t lo, int64_t hi) {
    for (int c = 0; c < n_cols; ++c) {
      const uint64_t* h = static_cast<const uint64_t*>(held_cols[c]);
      const uint64_t* f = static_cast<const uint64_t*>(fresh_cols[c]);
      uint64_t* o = static_cast<uint64_t*>(out_cols[c]);
      for (int64_t i = lo; i < hi; ++i) {
        const int64_t j = idx[i];
        o[i] = j < n_held ? h[j] : f[j - n_held];
      }
    }
  };
  const int nt = n_out < (1 << 16) ? 1 : static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  if (nt == 1) {
    work(0, n_out);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(work, n_out * t / nt, n_out * (t + 1) / nt);
    for (auto& x : th) x.join();
  }
  return PG_OK;
}

// out = concatenation of src[starts[i], starts[i] + lens[i]) for i < n (the held TOPK records'
// line prefixes, gathered from the per-batch prefix blobs at finalize).
int pg_gather_spans(const char* src, const int64_t* starts, const int64_t* lens, int64_t n, char* out) {
  PG_REQUIRE(n >= 0 && (n == 0 || (src && starts && lens && out)), PG_ERR_INVALID, "pg_gather_spans: bad arguments");
  char* o = out;
  for (int64_t i = 0; i < n; ++i) {
    std::memcpy(o, src + starts[i], static_cast<size_t>(lens[i]));
    o += lens[i];
  }
  return PG_OK;
}

}  // extern "C"
