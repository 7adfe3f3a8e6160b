// pg_ctx: the handle behind the C ABI (include/panelgwas_b200.h).
//
// One ctx per GPU. It owns the resident quantized panel, the per-batch device
// buffers (grow-only), a CUDA stream and timing events. A scan call runs, in
// stream order:  H2D (pitched) -> K1 stats -> K1 planes -> K2/K3 GEMM+epilogue
// -> candidate sort (cub radix, deterministic) -> K4 t/p.  Results stay on the
// device until fetched.
//
// Reference flow replaced (engine._run_scan_open / _process_batch,
// /root/reference/pkg/src/panelgwas/engine.py:178-219, 381-398).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "assoc.cuh"
#include "decode.cuh"
#include "panel.cuh"
#include "inflate.cuh"
#include "bgen_stage.cuh"
#include "pg_common.cuh"
#include "pstats.cuh"

namespace pg {
namespace {

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  int ensure(size_t n) {
    if (n <= cap && p != nullptr) return PG_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
      return PG_ERR_NOMEM;
    }
    cap = std::max<size_t>(n, 1);
    return PG_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

__global__ void count_skip_kernel(const int8_t* skip, int64_t m, unsigned long long* counts) {
  unsigned long long a = 0, b = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    a += skip[i] == 1;
    b += skip[i] == 2;
  }
  if (a) atomicAdd(counts, a);
  if (b) atomicAdd(counts + 1, b);
}

__global__ void row_map_kernel(const int8_t* skip, int64_t m, int64_t* new_row, unsigned long long* n_ok) {
  // single block, sequential-chunk scan: tiny (m ~ 1e4..1e5) and deterministic
  __shared__ long long part[1024];
  const int64_t per = (m + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = std::min<int64_t>(m, lo + per);
  long long c = 0;
  for (int64_t i = lo; i < hi; ++i) c += (skip[i] == 0);
  part[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (unsigned i = 0; i < blockDim.x; ++i) {
      const long long v = part[i];
      part[i] = run;
      run += v;
    }
    *n_ok = static_cast<unsigned long long>(run);
  }
  __syncthreads();
  long long base = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) new_row[i] = (skip[i] == 0) ? base++ : -1;
}

// contiguous rows (row_bytes apart) -> rows `pitch` bytes apart, 16-byte vector stores
__global__ void repitch_kernel(const uint8_t* __restrict__ src, int64_t row_bytes, uint8_t* __restrict__ dst,
                               int64_t pitch, int64_t m) {
  const int64_t row = blockIdx.x;
  const uint8_t* s = src + row * row_bytes;
  uint8_t* d = dst + row * pitch;
  for (int64_t c = threadIdx.x; c * 16 < pitch; c += blockDim.x) {
    uint8_t tmp[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t b = c * 16 + i;
      tmp[i] = b < row_bytes ? s[b] : 0;
    }
    *reinterpret_cast<uint4*>(d + c * 16) = *reinterpret_cast<const uint4*>(tmp);
  }
}

// Extension mode: V_res = V_u - sum_j w_j^2 with w = Q^T u_imp (side GEMM output),
// then the reference's post-projection variance / skip rule (kernel.py:409-417).
__global__ void resid_kernel(const double* __restrict__ w, int64_t ldw, int64_t n_cols, int64_t m,
                             const long long* __restrict__ n_miss, const long long* __restrict__ s_u,
                             const long long* __restrict__ ss_u, int64_t n_kept, double unit_scale, double* var,
                             int8_t* skip, double* invd_d, float* invd_f) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= m || skip[i] == 2) return;
  const long long n_obs = n_kept - n_miss[i];
  const __int128 nv = static_cast<__int128>(n_obs) * ss_u[i] - static_cast<__int128>(s_u[i]) * s_u[i];
  double v = static_cast<double>(nv) / static_cast<double>(n_obs);
  for (int64_t j = 0; j < n_cols; ++j) {
    const double x = w[i * ldw + j];
    v -= x * x;
  }
  const double vr = v / static_cast<double>(n_kept) * unit_scale * unit_scale;
  var[i] = vr;
  const bool mono = !(vr > 1e-12);
  skip[i] = mono ? 1 : 0;
  const double inv = mono ? __longlong_as_double(0x7ff8000000000000ll) : 1.0 / sqrt(static_cast<double>(n_kept) * v);
  invd_d[i] = inv;
  invd_f[i] = static_cast<float>(inv);
}

__global__ void rbar_kernel(const double* rbar_in, int64_t n, int64_t p_pad, float* rbar_out) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= p_pad) return;
  if (p >= n) {
    rbar_out[p] = __int_as_float(0x7f800000);  // +inf: padding phenotypes never match
    return;
  }
  // widen so the fp32 estimate never drops a pair whose exact fp64 |r| reaches the bar
  const double b = rbar_in[p];
  const double w = b * (1.0 - 1e-5) - 1e-7;
  rbar_out[p] = __double2float_rd(w);
}

}  // namespace
}  // namespace pg

namespace pg {
constexpr size_t kH2DBounce = size_t{64} << 20;  // pinned bounce buffers of upload_pageable (two)
}  // namespace pg

struct pg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

  // panel
  bool have_panel = false;
  int64_t n_src = 0, n_kept = 0, n_pheno = 0, p_pad = 0, k_pad = 0;
  pg::DBuf<int8_t> qh, q1, q0;
  pg::DBuf<double> scale_d, maxabs;
  pg::DBuf<float> scale_f, cq_f;
  pg::DBuf<long long> cq;
  pg::DBuf<int64_t> gidx;
  pg::DBuf<uint32_t> keep_bits;
  pg::DBuf<double> ystage;
  // device panel preparation (pg_ctx_prepare_panel -> pg_ctx_commit_panel)
  bool have_prepared = false;
  int64_t prep_rows = 0, prep_cols = 0;
  pg::DBuf<double> prep_q, prep_scratch, prep_mean, prep_centre, prep_sd;
  pg::DBuf<uint8_t> prep_flat;
  pg::DBuf<int> prep_bad;
  pg::DBuf<int64_t> colmap;
  // pipelined panel (pg_ctx_set_panel_async): phenotype column chunks are uploaded on
  // panel_copy and prepared + quantized on panel_prep; the first scan's GEMM waits for each
  // chunk in turn (chunk_ready) instead of for the whole panel
  cudaStream_t panel_copy = nullptr, panel_prep = nullptr;
  std::vector<cudaEvent_t> chunk_h2d, chunk_ready;
  std::vector<int64_t> chunk_pt;  // phenotype-tile boundaries, n_chunks + 1
  int64_t n_chunks = 0;
  // Chunk copies are issued lazily, at most two in flight: host-to-device copies run in
  // submission order across streams, so a batch staged after the panel call would otherwise
  // wait for the whole panel upload.
  int64_t chunk_issued = 0;
  int64_t async_chunk = 0, async_ld = 0, async_rank = 0;
  int64_t async_col0 = 0, async_col1 = 0;  // the columns this context prepares (all, or a rank's share)
  const double* async_y = nullptr;
  bool panel_pending = false;  // the compute stream has not yet waited for every chunk
  bool async_flags = false;    // zero-variance flags / sd / finiteness of the async panel on the device
  cudaEvent_t panel_ev = nullptr;
  cudaEvent_t geom_ev = nullptr;  // panel geometry (sample map) uploaded on panel_prep
  // A second context of the same job following this pipelined panel
  // (pg_ctx_follow_panel): each chunk, once prepared here, is copied to the follower's
  // buffers on its prep stream and marked ready there; the chunks are issued under pump_mu
  // by whichever of the two contexts needs the next one.
  pg_ctx* follower = nullptr;
  pg_ctx* leader = nullptr;
  std::mutex pump_mu;

  // scan parameters
  double df = 1.0;
  int mode = PG_MODE_THRESHOLD;
  bool have_scan = false;
  pg::DBuf<float> rbar;
  pg::DBuf<double> rbar_in;
  pg::DBuf<unsigned long long> max_abs_r;  // fp64 bits; tracked only when track_max_abs_r
  bool track_max_abs_r = false;

  // batch buffers
  pg::DBuf<uint8_t> packed;
  // pipelined staging: two device slots filled on a copy stream
  cudaStream_t copy_stream = nullptr;
  pg::DBuf<uint8_t> stage_buf[2];
  pg::DBuf<uint8_t> stage_raw[2];
  pg::DBuf<uint8_t> raw_rows;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  cudaEvent_t slot_free_ev[2] = {nullptr, nullptr};
  int stage_kind[2] = {-1, -1};
  // compressed BGEN staging (pg_stage_bgen): blob, block table, inflate scratch, checks
  pg::DBuf<uint8_t> bgen_blob[2], bgen_raw[2];
  pg::DBuf<int64_t> bgen_off[2], bgen_size[2], bgen_len[2];
  pg::DBuf<int> bgen_zstatus[2], bgen_bits[2];
  pg::DBuf<uint32_t> bgen_tok[2];  // two-phase GPU inflate: LZ77 tokens per stream
  pg::DBuf<int32_t> bgen_ntok[2];
  pg::DBuf<long long> bgen_diag[2];
  pg::DBuf<unsigned long long> bgen_summary[2];
  void* bgen_host[2] = {nullptr, nullptr};  // pinned copies of the validation summaries
  void* h2d_stage[2] = {nullptr, nullptr};   // pinned bounce buffers for large pageable uploads
  cudaEvent_t h2d_ev[2] = {nullptr, nullptr};
  int64_t bgen_pending[2] = {0, 0};         // batch size begun but not ended, per slot
  int64_t stage_m[2] = {0, 0};
  int64_t stage_pitch[2] = {0, 0};
  const uint8_t* stage_data[2] = {nullptr, nullptr};  // staged rows (stage_buf, or the inflated BGEN-8 blocks)
  int64_t stage_probs_off[2] = {0, 0};
  int64_t stage_ploidy_off[2] = {-1, -1};
  pg::DBuf<long long> n_miss, s_u, ss_u;
  pg::DBuf<double> sum_d, af, var, mu_d, invd_d;
  pg::DBuf<float> mu_f, invd_f;
  pg::DBuf<int8_t> skip;
  pg::DBuf<int> flags;
  pg::DBuf<int8_t> v, v127;
  pg::DBuf<unsigned long long> cand_key, cand_key_sorted;
  pg::DBuf<double> cand_r, cand_r_sorted, cand_t, cand_p;
  // effect sizes (pg_ctx_set_beta_scale): sd of each kept residualized phenotype, and the
  // candidates' beta / se
  bool beta_on = false;
  pg::DBuf<double> pheno_sd, cand_beta, cand_se;
  pg::DBuf<int64_t> cand_rows, cand_cols;
  pg::DBuf<unsigned long long> cand_count;
  pg::DBuf<unsigned long long> counters;  // [0] clamp, [1..2] skip counts, [3] n_ok
  pg::DBuf<uint8_t> sort_tmp;
  pg::DBuf<double> full_r;
  pg::DBuf<int64_t> new_row;
  pg::DBuf<uint8_t> full_out;
  pg::DBuf<double> scratch_a, scratch_b, scratch_c, scratch_d;
  pg::DBuf<long long> xacc, xacc_b;  // K-sliced runs (cohorts above kSliceK samples)
  // two-limb premask of PLINK THRESHOLD / TOPK scans (pg_ctx_set_two_limb_premask): ||q0_p||_2
  bool two_limb = true;
  bool q0n_valid = false;
  pg::DBuf<float> q0n;
  pg::DBuf<float4> mpack;
  pg::DBuf<long long> cand_xm;
  // F64 precision mode (pg_ctx_set_f64_panel): the panel's lo level + its partial sums
  bool f64_panel = false;
  pg::DBuf<int8_t> qh_lo, q1_lo, q0_lo;
  pg::DBuf<long long> cq_lo, xacc_lo, side_x_lo;
  // missing-call side path of the fused PLINK GEMM (pg_ctx_set_missing_side_gemm)
  bool side_missing = true;
  pg::DBuf<int> miss_flag, miss_prefix, miss_slot, miss_list, miss_count;
  pg::DBuf<int8_t> side_v, side_v127;
  pg::DBuf<long long> side_x;
  pg::DBuf<uint8_t> scan_tmp;

  // last batch
  int64_t last_m = 0, last_ncand = 0;
  int last_R = 1;
  int64_t cand_capacity = 0;
  unsigned long long cand_base = 0;  // test hook: initial candidate-counter value (pg_ctx_debug_candidate_base)
  bool fused_decode = true;
  bool wide_digits = true;
  // BGEN-8: transposed wide GEMM (A/B, PG_WIDE3T=1). Measured 9 % slower than kWide3 on C5
  // (4.56e9 vs 4.96-5.08e9 tests/s; no raster recovered it), so off by default.
  bool wide3t = false;

  // extension mode: quantized covariate basis (columns 1..rank-1) + side-GEMM output
  bool have_basis = false;
  int64_t basis_cols = 0;
  pg::DBuf<int8_t> bq_h, bq_1, bq_0;
  pg::DBuf<double> bscale_d, bmaxabs, bstage, wbuf;
  pg::DBuf<float> bscale_f, bcq_f;
  pg::DBuf<long long> bcq;
};

namespace pg {
namespace {

// Host rows -> pitched device rows: one bulk 1-D H2D (fast even for short, odd-sized
// rows, unlike a 2-D copy of 65k rows) into `raw`, then an on-device repitch.
int upload_rows(const void* host, int64_t m, int64_t row_bytes, int64_t pitch, pg::DBuf<uint8_t>& raw, uint8_t* dst,
                cudaStream_t s) {
  if (row_bytes == pitch) {
    PG_CUDA_CHECK(cudaMemcpyAsync(dst, host, static_cast<size_t>(m) * row_bytes, cudaMemcpyHostToDevice, s));
    return PG_OK;
  }
  PG_CHECK_STATUS(raw.ensure(static_cast<size_t>(m) * row_bytes));
  PG_CUDA_CHECK(cudaMemcpyAsync(raw.p, host, static_cast<size_t>(m) * row_bytes, cudaMemcpyHostToDevice, s));
  repitch_kernel<<<static_cast<unsigned>(m), 128, 0, s>>>(raw.p, row_bytes, dst, pitch, m);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int ctx_check(pg_ctx* c) {
  PG_REQUIRE(c != nullptr, PG_ERR_INVALID, "null pg_ctx");
  PG_CUDA_CHECK(cudaSetDevice(c->device));
  return PG_OK;
}

// Chunk j of leader c's pipelined panel -> follower f (pg_ctx_follow_panel): on f's prep
// stream, after the chunk is ready on c; then the chunk is ready on f as well.
int panel_copy_chunk(pg_ctx* c, pg_ctx* f, int64_t j) {
  const int64_t n_pheno = c->prep_cols, chunk = c->async_chunk;
  const int64_t c0 = c->async_col0 + j * chunk;
  const int64_t w = std::min(chunk, c->async_col1 - c0);
  const int64_t rows = c0 + w == n_pheno ? c->p_pad - c0 : w;
  const size_t off = static_cast<size_t>(c0) * c->k_pad, bytes = static_cast<size_t>(rows) * c->k_pad;
  cudaStream_t fs = f->panel_prep;
  PG_CUDA_CHECK(cudaStreamWaitEvent(fs, c->chunk_ready[j], 0));
  auto cp = [&](void* dst, const void* src, size_t n) -> int {
    PG_CUDA_CHECK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, fs));
    return PG_OK;
  };
  PG_CHECK_STATUS(cp(f->qh.p + off, c->qh.p + off, bytes));
  PG_CHECK_STATUS(cp(f->q1.p + off, c->q1.p + off, bytes));
  PG_CHECK_STATUS(cp(f->q0.p + off, c->q0.p + off, bytes));
  PG_CHECK_STATUS(cp(f->scale_d.p + c0, c->scale_d.p + c0, 8 * rows));
  PG_CHECK_STATUS(cp(f->scale_f.p + c0, c->scale_f.p + c0, 4 * rows));
  PG_CHECK_STATUS(cp(f->cq.p + c0, c->cq.p + c0, 8 * rows));
  PG_CHECK_STATUS(cp(f->cq_f.p + c0, c->cq_f.p + c0, 4 * rows));
  PG_CHECK_STATUS(cp(f->q0n.p + c0, c->q0n.p + c0, 4 * rows));
  if (c->f64_panel) {
    PG_CHECK_STATUS(cp(f->qh_lo.p + off, c->qh_lo.p + off, bytes));
    PG_CHECK_STATUS(cp(f->q1_lo.p + off, c->q1_lo.p + off, bytes));
    PG_CHECK_STATUS(cp(f->q0_lo.p + off, c->q0_lo.p + off, bytes));
    PG_CHECK_STATUS(cp(f->cq_lo.p + c0, c->cq_lo.p + c0, 8 * rows));
  }
  PG_CUDA_CHECK(cudaEventRecord(f->chunk_ready[j], fs));
  return PG_OK;
}

// Pipelined panel (pg_ctx_set_panel_async): enqueue chunk j — its H2D on panel_copy, then
// prepare + quantize + q0 norms on panel_prep, ending in chunk_ready[j].
int panel_issue(pg_ctx* c, int64_t j) {
  cudaStream_t ps = c->panel_prep, cs = c->panel_copy;
  const int64_t n_kept = c->prep_rows, n_pheno = c->prep_cols, chunk = c->async_chunk;
  const int64_t c0 = c->async_col0 + j * chunk;
  const int64_t w = std::min(chunk, c->async_col1 - c0);
  // panel rows (the padding rows past the last phenotype go with the last column)
  const int64_t rows = c0 + w == n_pheno ? c->p_pad - c0 : w;
  double* yj = c->ystage.p + static_cast<size_t>(n_kept) * (c0 - c->async_col0);  // the chunk as its own [n_kept, w]
  PG_CUDA_CHECK(cudaMemcpy2DAsync(yj, sizeof(double) * w, c->async_y + (c0 - c->async_col0),
                                  sizeof(double) * c->async_ld, sizeof(double) * w, n_kept, cudaMemcpyHostToDevice,
                                  cs));
  PG_CUDA_CHECK(cudaEventRecord(c->chunk_h2d[j], cs));
  PG_CUDA_CHECK(cudaStreamWaitEvent(ps, c->chunk_h2d[j], 0));
  pg::PanelPrepOut po;
  po.mean = c->prep_mean.p + c0;
  po.centre = c->prep_centre.p + c0;
  po.sd = c->prep_sd.p + c0;
  po.flat = c->prep_flat.p + c0;
  po.bad = c->prep_bad.p + j;
  PG_CHECK_STATUS(
      pg::panel_prepare(yj, n_kept, w, c->async_rank ? c->prep_q.p : nullptr, c->async_rank, c->prep_scratch.p, po, ps));
  // every column is kept (zero-variance ones quantize to 0): per column this is the
  // synchronous prepare + commit of all columns, bit for bit
  PanelPlanes pj;
  pj.qh = c->qh.p;
  pj.q1 = c->q1.p;
  pj.q0 = c->q0.p;
  const size_t off = static_cast<size_t>(c0) * c->k_pad;
  pj.qh += off;
  pj.q1 += off;
  pj.q0 += off;
  pj.scale_d = c->scale_d.p + c0;
  pj.scale_f = c->scale_f.p + c0;
  pj.cq = c->cq.p + c0;
  pj.cq_f = c->cq_f.p + c0;
  if (c->f64_panel) {
    pj.qh_lo = c->qh_lo.p + off;
    pj.q1_lo = c->q1_lo.p + off;
    pj.q0_lo = c->q0_lo.p + off;
    pj.cq_lo = c->cq_lo.p + c0;
  }
  PG_CHECK_STATUS(panel_quantize(yj, n_kept, w, w, nullptr, c->gidx.p, c->k_pad, rows, pj, c->maxabs.p + c0, ps));
  PG_CHECK_STATUS(panel_q0_norms(c->q0.p + off, rows, c->k_pad, c->q0n.p + c0, ps));
  PG_CUDA_CHECK(cudaEventRecord(c->chunk_ready[j], ps));
  if (c->follower != nullptr) PG_CHECK_STATUS(panel_copy_chunk(c, c->follower, j));
  return PG_OK;
}

// Issue chunks up to `upto` (inclusive), keeping at most two chunk copies in flight
// (blocks the host on an earlier chunk's copy when needed); upto < 0: only as many as can
// be issued without blocking.
int panel_pump(pg_ctx* c, int64_t upto) {
  if (c->leader != nullptr) return panel_pump(c->leader, upto);  // the leader issues for both
  std::lock_guard<std::mutex> lock(c->pump_mu);
  while (c->chunk_issued < c->n_chunks) {
    const int64_t j = c->chunk_issued;
    if (j >= 2) {
      if (j > upto) {
        const cudaError_t q = cudaEventQuery(c->chunk_h2d[j - 2]);
        if (q == cudaErrorNotReady) break;
        PG_CUDA_CHECK(q);
      } else {
        PG_CUDA_CHECK(cudaEventSynchronize(c->chunk_h2d[j - 2]));
      }
    } else if (j > upto && upto >= 0) {
      break;
    }
    PG_CHECK_STATUS(panel_issue(c, j));
    ++c->chunk_issued;
  }
  return PG_OK;
}

// A pipelined panel still being prepared: `s` waits for every chunk (work that reads the
// whole panel), after which the panel is an ordinary resident panel for that stream.
int panel_wait_all(pg_ctx* c, cudaStream_t s) {
  if (c->panel_pending) {
    PG_CHECK_STATUS(panel_pump(c, c->n_chunks - 1));
    PG_CUDA_CHECK(cudaStreamWaitEvent(s, c->chunk_ready[c->n_chunks - 1], 0));
    c->panel_pending = false;
  }
  return PG_OK;
}

// Before a new panel replaces the current one: no pipelined preparation may still write it.
int panel_drain(pg_ctx* c) {
  if (c->panel_prep) {
    if (c->leader == nullptr || c->panel_pending) PG_CHECK_STATUS(panel_pump(c, c->n_chunks - 1));
    PG_CUDA_CHECK(cudaStreamSynchronize(c->panel_prep));
  }
  if (c->follower != nullptr) {  // every chunk was issued (and copied): release the follower
    PG_CUDA_CHECK(cudaStreamSynchronize(c->follower->panel_prep));
    c->follower->chunk_issued = c->follower->n_chunks;
    c->follower->leader = nullptr;
    c->follower = nullptr;
  }
  if (c->leader != nullptr) {
    c->leader->follower = nullptr;
    c->leader = nullptr;
    c->chunk_issued = c->n_chunks;
  }
  c->panel_pending = false;
  c->async_flags = false;
  c->async_y = nullptr;
  return PG_OK;
}

// Panel geometry, keep bits and limb buffers (shared by the synchronous and pipelined
// uploads); the small index uploads go on `s`.
int panel_geometry(pg_ctx* c, int64_t n_kept, int64_t n_pheno, int64_t n_src, const int64_t* h_gidx, cudaStream_t s,
                   PanelPlanes& pp) {
  PG_REQUIRE(n_kept >= 1 && n_pheno >= 1 && n_src >= n_kept, PG_ERR_INVALID,
             "invalid panel geometry n_kept=%lld n_pheno=%lld n_src=%lld", (long long)n_kept, (long long)n_pheno,
             (long long)n_src);
  std::vector<uint32_t> bits;
  c->n_src = n_src;
  c->n_kept = n_kept;
  c->n_pheno = n_pheno;
  c->p_pad = round_up(n_pheno, kTileP);
  PG_REQUIRE(round_up(n_src, 64) <= (int64_t(1) << 30), PG_ERR_CONFIG, "%lld genotype samples: too many",
             (long long)n_src);
  c->k_pad = round_up(n_src, 64);
  bits.assign(c->k_pad / 32 + 1, 0u);
  for (int64_t i = 0; i < n_kept; ++i) {
    const int64_t g = h_gidx[i];
    PG_REQUIRE(g >= 0 && g < n_src, PG_ERR_INVALID, "geno_row_index out of range");
    PG_REQUIRE(((bits[g >> 5] >> (g & 31)) & 1u) == 0, PG_ERR_INVALID, "duplicate geno_row_index %lld",
               (long long)g);
    bits[g >> 5] |= 1u << (g & 31);
  }
  const size_t plane = static_cast<size_t>(c->p_pad) * c->k_pad;
  PG_CHECK_STATUS(c->qh.ensure(plane));
  PG_CHECK_STATUS(c->q1.ensure(plane));
  PG_CHECK_STATUS(c->q0.ensure(plane));
  PG_CHECK_STATUS(c->scale_d.ensure(c->p_pad));
  PG_CHECK_STATUS(c->scale_f.ensure(c->p_pad));
  PG_CHECK_STATUS(c->cq.ensure(c->p_pad));
  PG_CHECK_STATUS(c->cq_f.ensure(c->p_pad));
  PG_CHECK_STATUS(c->maxabs.ensure(c->p_pad));
  PG_CHECK_STATUS(c->gidx.ensure(n_kept));
  PG_CHECK_STATUS(c->keep_bits.ensure(bits.size()));
  // pageable sources: both copies are complete (staged) when the calls return
  PG_CUDA_CHECK(cudaMemcpyAsync(c->gidx.p, h_gidx, sizeof(int64_t) * n_kept, cudaMemcpyHostToDevice, s));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->keep_bits.p, bits.data(), sizeof(uint32_t) * bits.size(), cudaMemcpyHostToDevice, s));
  pp = PanelPlanes{};
  pp.qh = c->qh.p;
  pp.q1 = c->q1.p;
  pp.q0 = c->q0.p;
  pp.scale_d = c->scale_d.p;
  pp.scale_f = c->scale_f.p;
  pp.cq = c->cq.p;
  pp.cq_f = c->cq_f.p;
  if (c->f64_panel) {
    PG_CHECK_STATUS(c->qh_lo.ensure(plane));
    PG_CHECK_STATUS(c->q1_lo.ensure(plane));
    PG_CHECK_STATUS(c->q0_lo.ensure(plane));
    PG_CHECK_STATUS(c->cq_lo.ensure(c->p_pad));
    pp.qh_lo = c->qh_lo.p;
    pp.q1_lo = c->q1_lo.p;
    pp.q0_lo = c->q0_lo.p;
    pp.cq_lo = c->cq_lo.p;
  }
  c->q0n_valid = false;
  return PG_OK;
}

int upload_panel_common(pg_ctx* c, const double* d_y, int64_t n_kept, int64_t n_pheno, int64_t ld,
                        const int64_t* h_gidx, int64_t n_src, const int64_t* d_cols = nullptr) {
  PG_REQUIRE(ld >= n_pheno, PG_ERR_INVALID, "invalid panel leading dimension %lld < %lld", (long long)ld,
             (long long)n_pheno);
  PG_CHECK_STATUS(panel_drain(c));
  PanelPlanes pp;
  PG_CHECK_STATUS(panel_geometry(c, n_kept, n_pheno, n_src, h_gidx, c->stream, pp));
  PG_CHECK_STATUS(
      panel_quantize(d_y, n_kept, n_pheno, ld, d_cols, c->gidx.p, c->k_pad, c->p_pad, pp, c->maxabs.p, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->have_panel = true;
  c->have_scan = false;
  c->have_basis = false;
  c->beta_on = false;  // phenotype scales belong to the previous panel's columns
  return PG_OK;
}

int64_t expected_row_bytes(int kind, int64_t n_src) {
  switch (kind) {
    case PG_GENO_BED: return (n_src + 3) / 4;
    case PG_GENO_BGEN8: return n_src * 3;
    case PG_GENO_BGEN16: return n_src * 5;
    case PG_GENO_DENSE_F64: return n_src * 8;
    default: return -1;
  }
}

// Largest candidate count of one batch: the cub sort takes int item counts, and 2^30 pairs
// already hold ~70 GB of device candidate buffers.
constexpr int64_t kMaxCandidates = int64_t(1) << 30;
// Largest side-GEMM output (8 B per marker-with-missing-calls x phenotype) before a batch
// falls back to the two-row planes path.
constexpr int64_t kSideBytesMax = int64_t(12) << 30;

int scan_common(pg_ctx* c, int kind, const uint8_t* d_data, int64_t m, int64_t pitch, pg_batch_info* info,
                int64_t probs_off = 0, int64_t ploidy_off = -1) {
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_scan: no panel uploaded (pg_ctx_set_panel)");
  PG_REQUIRE(c->have_scan, PG_ERR_STATE, "pg_scan: scan parameters not set (pg_ctx_set_scan)");
  PG_REQUIRE(m >= 1, PG_ERR_INVALID, "pg_scan: empty batch");
  cudaStream_t s = c->stream;
  PG_CUDA_CHECK(cudaEventRecord(c->ev[0], s));

  GenoBlock b;
  b.kind = kind;
  b.data = d_data;
  b.pitch = pitch;
  b.n_markers = m;
  b.n_src = c->n_src;
  b.n_kept = c->n_kept;
  b.keep_bits = c->keep_bits.p;
  b.all_kept = c->n_kept == c->n_src ? 1 : 0;
  b.probs_off = probs_off;
  b.ploidy_off = ploidy_off;

  // marker slots for any tiling: ternary tiles hold 256 / R markers, wide tiles 40
  const int64_t m_cap = round_up(m, 256) + 256;
  PG_CHECK_STATUS(c->flags.ensure(2));
  PG_CUDA_CHECK(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 2, s));
  int hflags[2] = {0, 0};
  if (kind == PG_GENO_DENSE_F64) {
    MarkerStats tmp;
    tmp.flags = c->flags.p;
    PG_CHECK_STATUS(geno_check_integral(b, tmp, s));
    PG_CUDA_CHECK(cudaMemcpyAsync(hflags, c->flags.p, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
    PG_CUDA_CHECK(cudaStreamSynchronize(s));
    b.dense_real = hflags[1] != 0;
  }
  for (auto* buf : {&c->n_miss, &c->s_u, &c->ss_u}) PG_CHECK_STATUS(buf->ensure(m_cap));
  for (auto* buf : {&c->sum_d, &c->af, &c->var, &c->mu_d, &c->invd_d}) PG_CHECK_STATUS(buf->ensure(m_cap));
  PG_CHECK_STATUS(c->mu_f.ensure(m_cap));
  PG_CHECK_STATUS(c->invd_f.ensure(m_cap));
  PG_CHECK_STATUS(c->skip.ensure(m_cap));
  MarkerStats st;
  st.n_miss = c->n_miss.p;
  st.s_u = c->s_u.p;
  st.ss_u = c->ss_u.p;
  st.sum_d = c->sum_d.p;
  st.af = c->af.p;
  st.var = c->var.p;
  st.skip = c->skip.p;
  st.mu_d = c->mu_d.p;
  st.mu_f = c->mu_f.p;
  st.invd_d = c->invd_d.p;
  st.invd_f = c->invd_f.p;
  st.flags = c->flags.p;
  PG_CHECK_STATUS(geno_stats(b, st, m_cap, s));
  // PLINK batches with missing calls: only the markers that have them carry a mask row, in
  // a side GEMM; the batch keeps the fused one-row-per-marker GEMM (K-sliced and extension
  // runs use the two-row planes instead)
  const bool side_ok = c->side_missing && c->fused_decode && kind == PG_GENO_BED && c->k_pad <= kSliceK &&
                       !c->have_basis;
  int n_side = 0;
  if (side_ok) {
    for (auto* buf : {&c->miss_flag, &c->miss_prefix, &c->miss_list}) PG_CHECK_STATUS(buf->ensure(m));
    PG_CHECK_STATUS(c->miss_slot.ensure(m_cap));
    PG_CHECK_STATUS(c->miss_count.ensure(1));
    PG_CUDA_CHECK(cudaMemsetAsync(c->miss_slot.p, 0xFF, sizeof(int) * m_cap, s));  // -1: no missing calls
    PG_CHECK_STATUS(missing_flags(c->n_miss.p, c->skip.p, m, c->miss_flag.p, s));
    size_t tmp_bytes = 0;
    PG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, c->miss_flag.p, c->miss_prefix.p,
                                                static_cast<int>(m), s));
    PG_CHECK_STATUS(c->scan_tmp.ensure(tmp_bytes));
    PG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(c->scan_tmp.p, tmp_bytes, c->miss_flag.p, c->miss_prefix.p,
                                                static_cast<int>(m), s));
    PG_CHECK_STATUS(missing_slot_map(c->miss_flag.p, c->miss_prefix.p, m, c->miss_slot.p, c->miss_list.p,
                                     c->miss_count.p, s));
    PG_CUDA_CHECK(cudaMemcpyAsync(&n_side, c->miss_count.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  // the row layout depends on the batch's missing calls only for PLINK / integral dense rows;
  // wide-digit batches (BGEN, real dense) go on to the GEMM without a host round trip
  if (!(c->wide_digits && geno_wide(b)) || side_ok) {
    PG_CUDA_CHECK(cudaMemcpyAsync(hflags, c->flags.p, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
    PG_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // dosage sources use the wide-digit GEMM (3 rows per BGEN-8 marker, 4 otherwise) unless
  // disabled for A/B tests
  int R = geno_rows_per_marker(b, hflags[0] != 0, c->wide_digits);
  const int64_t side_rows = round_up(n_side, kTileC);
  const bool use_side = side_ok && R == 2 && side_rows * c->p_pad * 8 <= kSideBytesMax;
  if (use_side) R = 1;
  const bool wide = R == kWideRows || R == kWideRows3;
  // BGEN-8: the transposed wide GEMM (genotype rows as A) unless the run needs K slices,
  // the extension-mode side GEMM or the per-phenotype max |r| (kept on the kWide3 kernel)
  const bool wide3t = R == kWideRows3 && c->wide3t && c->k_pad <= kSliceK && !c->have_basis && !c->track_max_abs_r &&
                      !c->f64_panel;
  // PLINK rows without missing calls: the GEMM decodes the packed codes itself
  const bool fused = c->fused_decode && kind == PG_GENO_BED && R == 1;
  // THRESHOLD / TOPK: two MMAs per 32 samples (the q0 limb deferred to the candidates), for the
  // fused PLINK GEMM and the BGEN-8 wide GEMM (whose tile then widens to 240 rows)
  const bool two_limb_ok =
      c->two_limb && c->mode != PG_MODE_FULL && !c->track_max_abs_r && c->k_pad <= kSliceK && !c->f64_panel;
  const bool wide_two = two_limb_ok && (R == kWideRows3 || R == kWideRows) && !wide3t && !c->have_basis;
  const bool two_limb = two_limb_ok && (fused || wide_two);
  const int64_t c_pad =
      wide3t ? round_up((m + 9) / 10 * 32, kTileC)
             : round_up(m * R, wide ? (R == kWideRows3 ? (wide_two ? kTileCWide3Two : kTileCWide3)
                                                        : (wide_two ? kTileC : kTileCWide))
                                    : kTileC);
  if (two_limb && !c->q0n_valid) {
    PG_CHECK_STATUS(c->q0n.ensure(c->p_pad));
    PG_CHECK_STATUS(panel_q0_norms(c->q0.p, c->p_pad, c->k_pad, c->q0n.p, s));
    c->q0n_valid = true;
  }
  int64_t launches = (kind == PG_GENO_DENSE_F64 ? 2 : 1);
  if (!fused) {
    PG_CHECK_STATUS(c->v.ensure(static_cast<size_t>(c_pad) * c->k_pad));
    if (!wide) PG_CHECK_STATUS(c->v127.ensure(static_cast<size_t>(c_pad) * c->k_pad));
    PG_CHECK_STATUS(geno_planes(b, R, c->v.p, wide ? nullptr : c->v127.p, c_pad, c->k_pad, s, wide3t));
    ++launches;
  }
  auto run_gemm_on = [&](const AssocEpilogue& e, const int8_t* a, const int8_t* b1, const int8_t* b0,
                         int64_t pp) -> int {
    if (fused) return launch_assoc_packed(a, b1, b0, pp, d_data, pitch, m, c->k_pad, e, s);
    if (wide3t) return launch_assoc_wide3t(a, b1, b0, pp, c->v.p, c_pad, c->k_pad, e, s);
    if (wide) return launch_assoc_wide(a, b1, b0, pp, c->v.p, c_pad, c->k_pad, e, s);
    return launch_assoc(a, b1, b0, pp, c->v.p, c->v127.p, c_pad, c->k_pad, e, s);
  };
  // side GEMM over the mask rows of the markers with missing calls -> Mq per (marker, phenotype)
  bool side_pending = use_side && n_side > 0;
  if (side_pending) {
    PG_CHECK_STATUS(c->side_v.ensure(static_cast<size_t>(side_rows) * c->k_pad));
    PG_CHECK_STATUS(c->side_v127.ensure(static_cast<size_t>(side_rows) * c->k_pad));
    PG_CHECK_STATUS(c->side_x.ensure(static_cast<size_t>(side_rows) * c->p_pad));
    if (c->f64_panel) PG_CHECK_STATUS(c->side_x_lo.ensure(static_cast<size_t>(side_rows) * c->p_pad));
    PG_CHECK_STATUS(missing_mask_planes(b, c->miss_list.p, n_side, c->side_v.p, c->side_v127.p, side_rows, c->k_pad, s));
    ++launches;
  }
  // one side GEMM per panel level (hi, and lo in F64 mode), run once per batch
  bool side_done[2] = {false, false};
  auto run_side = [&](int level) -> int {
    if (!side_pending || side_done[level]) return PG_OK;
    side_done[level] = true;
    PG_CHECK_STATUS(panel_wait_all(c, s));
    AssocEpilogue es{};
    es.rows_per_marker = 1;
    es.m_valid = n_side;
    es.p_valid = c->n_pheno;
    es.mu_f = c->mu_f.p;
    es.mu_d = c->mu_d.p;
    es.invd_f = c->invd_f.p;
    es.invd_d = c->invd_d.p;
    es.scale_f = c->scale_f.p;
    es.scale_d = c->scale_d.p;
    es.cq_f = c->cq_f.p;
    es.cq = c->cq.p;
    es.side_ld = c->p_pad;
    if (two_limb) es.q0n = c->q0n.p;  // two-limb scans: the side GEMM defers q0 as well
    ++launches;
    if (level == 1) {  // side_x_lo was sized with the other side buffers (its pointer is already in use)
      es.side_out = c->side_x_lo.p;
      return launch_assoc(c->qh_lo.p, c->q1_lo.p, c->q0_lo.p, c->p_pad, c->side_v.p, c->side_v127.p, side_rows,
                          c->k_pad, es, s);
    }
    es.side_out = c->side_x.p;
    return launch_assoc(c->qh.p, c->q1.p, c->q0.p, c->p_pad, c->side_v.p, c->side_v127.p, side_rows, c->k_pad, es, s);
  };
  auto run_gemm = [&](const AssocEpilogue& e) -> int {
    if (c->f64_panel) {
      PG_CHECK_STATUS(panel_wait_all(c, s));
      // lo level first (partials only), then the hi level, whose statistics add the lo partials
      AssocEpilogue el = e;
      el.x_accum = c->xacc_lo.p;
      el.x_partials_only = 1;
      el.x_lo = nullptr;
      if (e.side_slot) el.side_x = c->side_x_lo.p;
      PG_CHECK_STATUS(run_side(1));
      PG_CHECK_STATUS(run_gemm_on(el, c->qh_lo.p, c->q1_lo.p, c->q0_lo.p, c->p_pad));
      ++launches;
      AssocEpilogue eh = e;
      eh.x_lo = c->xacc_lo.p;
      PG_CHECK_STATUS(run_side(0));
      return run_gemm_on(eh, c->qh.p, c->q1.p, c->q0.p, c->p_pad);
    }
    PG_CHECK_STATUS(run_side(0));
    if (c->panel_pending && !wide3t && e.x_accum == nullptr) {
      // pipelined panel: one launch per phenotype chunk, each as soon as its chunk is ready,
      // so the first batch's GEMM overlaps the upload of the later chunks
      for (int64_t j = 0; j < c->n_chunks; ++j) {
        PG_CHECK_STATUS(panel_pump(c, j));
        PG_CUDA_CHECK(cudaStreamWaitEvent(s, c->chunk_ready[j], 0));
        AssocEpilogue ej = e;
        ej.pt_base = static_cast<int>(c->chunk_pt[j]);
        ej.pt_count = static_cast<int>(c->chunk_pt[j + 1] - c->chunk_pt[j]);
        PG_CHECK_STATUS(run_gemm_on(ej, c->qh.p, c->q1.p, c->q0.p, c->p_pad));
        if (j) ++launches;
      }
      c->panel_pending = false;
      return PG_OK;
    }
    PG_CHECK_STATUS(panel_wait_all(c, s));
    return run_gemm_on(e, c->qh.p, c->q1.p, c->q0.p, c->p_pad);
  };
  if (c->have_basis) {
    PG_CHECK_STATUS(panel_wait_all(c, s));
    // K5: w = Q^T u_imp for every marker (exact side GEMM against the quantized basis)
    PG_CHECK_STATUS(c->wbuf.ensure(static_cast<size_t>(c_pad / R) * kTileP));
    PG_CHECK_STATUS(c->cand_count.ensure(1));
    AssocEpilogue eb{};
    eb.rows_per_marker = R;
    eb.raw = 1;
    eb.m_valid = m;
    eb.p_valid = c->basis_cols;
    eb.mu_f = c->mu_f.p;
    eb.mu_d = c->mu_d.p;
    eb.invd_f = c->invd_f.p;
    eb.invd_d = c->invd_d.p;
    eb.scale_f = c->bscale_f.p;
    eb.scale_d = c->bscale_d.p;
    eb.cq_f = c->bcq_f.p;
    eb.cq = c->bcq.p;
    eb.rbar = nullptr;
    eb.cand_count = c->cand_count.p;
    eb.full_r = c->wbuf.p;
    eb.full_ld = kTileP;
    if (c->k_pad > kSliceK) {  // more samples than one exact int32 slice
      PG_CHECK_STATUS(c->xacc_b.ensure(static_cast<size_t>(c_pad / R) * kTileP * 2));
      eb.x_accum = c->xacc_b.p;
      eb.x_ld = kTileP;
    }
    PG_CHECK_STATUS(run_gemm_on(eb, c->bq_h.p, c->bq_1.p, c->bq_0.p, kTileP));
    resid_kernel<<<static_cast<unsigned>((m + 255) / 256), 256, 0, s>>>(
        c->wbuf.p, kTileP, c->basis_cols, m, c->n_miss.p, c->s_u.p, c->ss_u.p, c->n_kept, geno_unit_scale(b),
        c->var.p, c->skip.p, c->invd_d.p, c->invd_f.p);
    PG_CUDA_CHECK(cudaGetLastError());
    launches += 2;
  }
  float decode_ms = 0.f;

  PG_CHECK_STATUS(c->counters.ensure(4));
  PG_CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, sizeof(unsigned long long) * 4, s));
  count_skip_kernel<<<64, 256, 0, s>>>(c->skip.p, m, c->counters.p + 1);
  PG_CUDA_CHECK(cudaGetLastError());
  ++launches;
  PG_CUDA_CHECK(cudaEventRecord(c->ev[1], s));

  AssocEpilogue ep{};
  ep.rows_per_marker = R;
  ep.m_valid = m;
  ep.p_valid = c->n_pheno;
  ep.mu_f = c->mu_f.p;
  ep.mu_d = c->mu_d.p;
  ep.invd_f = c->invd_f.p;
  ep.invd_d = c->invd_d.p;
  ep.scale_f = c->scale_f.p;
  ep.scale_d = c->scale_d.p;
  ep.cq_f = c->cq_f.p;
  ep.cq = c->cq.p;
  ep.max_abs_r = c->track_max_abs_r ? c->max_abs_r.p : nullptr;
  if (use_side && n_side > 0) {
    ep.side_x = c->side_x.p;
    ep.side_slot = c->miss_slot.p;
    ep.side_ld = c->p_pad;
    ep.side_two = two_limb ? 1 : 0;
  }
  if (two_limb) {
    ep.q0n = c->q0n.p;
    PG_CHECK_STATUS(c->mpack.ensure(m_cap));  // m_cap covers every marker slot of the tiles
    PG_CHECK_STATUS(pack_marker_terms(c->mu_f.p, c->mu_d.p, c->invd_f.p, c->ss_u.p, c->n_miss.p, m_cap, c->mpack.p, s));
    ep.mpack = c->mpack.p;
    ++launches;
  }
  PG_CHECK_STATUS(c->cand_count.ensure(1));
  ep.cand_count = c->cand_count.p;
  // exact int64 partials per (marker, phenotype): K-sliced contraction, and / or the two
  // panel levels of the F64 precision mode
  if (c->k_pad > kSliceK || c->f64_panel) {
    PG_CHECK_STATUS(c->xacc.ensure(static_cast<size_t>(c_pad / R) * c->p_pad * 2));
    ep.x_accum = c->xacc.p;
    ep.x_ld = c->p_pad;
  }
  if (c->f64_panel) {
    PG_CHECK_STATUS(c->xacc_lo.ensure(static_cast<size_t>(c_pad / R) * c->p_pad * 2));
    ep.cq_lo = c->cq_lo.p;
  }
  int64_t ncand = 0;
  if (c->mode == PG_MODE_FULL) {
    PG_CHECK_STATUS(c->full_r.ensure(static_cast<size_t>(c_pad / R) * c->p_pad));
    ep.full_r = c->full_r.p;
    ep.full_ld = c->p_pad;
    ep.rbar = nullptr;
    ep.cand_cap = 0;
    PG_CUDA_CHECK(cudaMemsetAsync(c->cand_count.p, 0, sizeof(unsigned long long), s));
    PG_CUDA_CHECK(cudaEventRecord(c->ev[1], s));
    PG_CHECK_STATUS(run_gemm(ep));
    PG_CUDA_CHECK(cudaEventRecord(c->ev[2], s));
    ++launches;
  } else {
    ep.rbar = c->rbar.p;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (c->cand_capacity < 1024) {
        PG_CHECK_STATUS(c->cand_key.ensure(1 << 20));
        PG_CHECK_STATUS(c->cand_r.ensure(1 << 20));
        c->cand_capacity = 1 << 20;
      }
      if (wide_two) PG_CHECK_STATUS(c->cand_xm.ensure(c->cand_capacity));
      ep.cand_key = c->cand_key.p;
      ep.cand_r = c->cand_r.p;
      ep.cand_xm = wide_two ? c->cand_xm.p : nullptr;
      ep.cand_cap = c->cand_capacity;
      ep.cand_base = c->cand_base;
      // the 64-bit counter starts at cand_base (0 except under the test hook); slots are
      // counter - cand_base, so a count that crosses 2^31 inside a launch stays exact
      PG_CUDA_CHECK(cudaMemcpyAsync(c->cand_count.p, &c->cand_base, sizeof(unsigned long long),
                                    cudaMemcpyHostToDevice, s));
      PG_CUDA_CHECK(cudaEventRecord(c->ev[1], s));
      PG_CHECK_STATUS(run_gemm(ep));
      PG_CUDA_CHECK(cudaEventRecord(c->ev[2], s));
      ++launches;
      unsigned long long hcount = 0;
      PG_CUDA_CHECK(cudaMemcpyAsync(&hcount, c->cand_count.p, sizeof(hcount), cudaMemcpyDeviceToHost, s));
      PG_CUDA_CHECK(cudaStreamSynchronize(s));
      ncand = static_cast<int64_t>(hcount - c->cand_base);
      if (ncand <= c->cand_capacity) break;
      // overflow: grow to fit and recompute (results are order-independent after the sort).
      // Growth is bounded: the sort takes int item counts and every candidate costs ~64 B of
      // device buffers, so a batch whose premask admits more than kMaxCandidates pairs is an
      // error the caller fixes with smaller batches (engine.device_batch_size bounds it).
      PG_REQUIRE(ncand <= kMaxCandidates, PG_ERR_CONFIG,
                 "pg_scan: %lld candidate pairs in one batch of %lld markers exceed the limit of %lld; "
                 "scan smaller batches (expected candidates ~ p_threshold x markers x phenotypes)",
                 (long long)ncand, (long long)m, (long long)kMaxCandidates);
      const int64_t newcap = ncand + ncand / 8 + 1024;
      PG_CHECK_STATUS(c->cand_key.ensure(newcap));
      PG_CHECK_STATUS(c->cand_r.ensure(newcap));
      c->cand_capacity = newcap;  // max |r| is idempotent under recomputation
    }
  }

  if (ncand > 0 && two_limb) {
    // candidates hold X' = X - sum q0 u: add the deferred limb exactly, then r in fp64
    if (wide_two)
      PG_CHECK_STATUS(refine_wide_two(c->cand_key.p, c->cand_r.p, c->cand_xm.p, ncand, c->v.p, c->q0.p, c->k_pad, ep, s));
    else
      PG_CHECK_STATUS(refine_two_limb(c->cand_key.p, c->cand_r.p, ncand, d_data, pitch, c->q0.p, c->k_pad, ep, s));
    ++launches;
  }
  if (ncand > 0) {
    PG_CHECK_STATUS(c->cand_key_sorted.ensure(ncand));
    PG_CHECK_STATUS(c->cand_r_sorted.ensure(ncand));
    PG_CHECK_STATUS(c->cand_t.ensure(ncand));
    PG_CHECK_STATUS(c->cand_p.ensure(ncand));
    PG_CHECK_STATUS(c->cand_rows.ensure(ncand));
    PG_CHECK_STATUS(c->cand_cols.ensure(ncand));
    int end_bit = 32;
    while (end_bit < 64 && (1ull << (end_bit - 32)) <= static_cast<unsigned long long>(m)) ++end_bit;
    size_t tmp_bytes = 0;
    PG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, c->cand_key.p, c->cand_key_sorted.p,
                                                  c->cand_r.p, c->cand_r_sorted.p, ncand, 0, end_bit, s));
    PG_CHECK_STATUS(c->sort_tmp.ensure(tmp_bytes));
    PG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(c->sort_tmp.p, tmp_bytes, c->cand_key.p, c->cand_key_sorted.p,
                                                  c->cand_r.p, c->cand_r_sorted.p, ncand, 0, end_bit, s));
    BetaArgs beta;
    if (c->beta_on) {
      PG_CHECK_STATUS(c->cand_beta.ensure(ncand));
      PG_CHECK_STATUS(c->cand_se.ensure(ncand));
      beta.var_m = c->var.p;
      beta.sd_p = c->pheno_sd.p;
      beta.beta = c->cand_beta.p;
      beta.se = c->cand_se.p;
    }
    PG_CHECK_STATUS(finalize_candidates(c->cand_key_sorted.p, c->cand_r_sorted.p, ncand, c->df, c->cand_rows.p,
                                        c->cand_cols.p, c->cand_r_sorted.p, c->cand_t.p, c->cand_p.p, c->counters.p,
                                        beta, s));
    ++launches;
  }
  PG_CUDA_CHECK(cudaEventRecord(c->ev[3], s));
  unsigned long long hc[4] = {0, 0, 0, 0};
  PG_CUDA_CHECK(cudaMemcpyAsync(hc, c->counters.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
  PG_CUDA_CHECK(cudaStreamSynchronize(s));
  c->last_m = m;
  c->last_ncand = ncand;
  c->last_R = R;
  if (info) {
    info->n_markers = m;
    info->n_candidates = ncand;
    info->clamp_count = static_cast<int64_t>(hc[0]);
    info->n_skipped_monomorphic = static_cast<int64_t>(hc[1]);
    info->n_skipped_all_missing = static_cast<int64_t>(hc[2]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    info->decode_ms = ms + decode_ms;
    cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]);
    info->gemm_ms = ms;
    info->launches = launches;
    info->rows_per_marker = R;
  }
  return PG_OK;
}

}  // namespace
}  // namespace pg

using namespace pg;

extern "C" {

int pg_ctx_create(int device, pg_ctx** out) {
  PG_REQUIRE(out != nullptr, PG_ERR_INVALID, "pg_ctx_create: null out");
  *out = nullptr;
  int n = 0;
  PG_CUDA_CHECK(cudaGetDeviceCount(&n));
  PG_REQUIRE(device >= 0 && device < n, PG_ERR_CUDA, "no CUDA device %d (%d visible)", device, n);
  cudaDeviceProp prop;
  PG_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  PG_REQUIRE(prop.major == 10 && prop.minor == 0, PG_ERR_CUDA,
             "device %d is sm_%d%d; panelgwas_b200 kernels are built for sm_100a (B200) only", device, prop.major,
             prop.minor);
  PG_CUDA_CHECK(cudaSetDevice(device));
  pg_ctx* c = new pg_ctx();
  c->device = device;
  if (const char* e = std::getenv("PG_WIDE3T")) c->wide3t = std::atoi(e) != 0;
  if (const char* e = std::getenv("PG_TWO_LIMB")) c->two_limb = std::atoi(e) != 0;
  PG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  PG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  for (auto& e : c->ev) PG_CUDA_CHECK(cudaEventCreate(&e));
  for (int i = 0; i < 2; ++i) {
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&c->slot_free_ev[i], cudaEventDisableTiming));
    // the pageable-upload bounce buffers are page-locked now (contexts are created while the
    // host parses tables), not on the first panel upload
    PG_CUDA_CHECK(cudaHostAlloc(&c->h2d_stage[i], pg::kH2DBounce, cudaHostAllocDefault));
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&c->h2d_ev[i], cudaEventDisableTiming));
  }
  *out = c;
  return PG_OK;
}

int pg_ctx_destroy(pg_ctx* c) {
  if (c == nullptr) return PG_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->follower) {  // chunks not issued yet will never reach the follower
    if (c->chunk_issued < c->n_chunks) c->follower->have_panel = false;
    c->follower->chunk_issued = c->follower->n_chunks;
    c->follower->leader = nullptr;
  }
  if (c->leader) c->leader->follower = nullptr;
  if (c->panel_prep) {
    cudaStreamSynchronize(c->panel_prep);
    cudaStreamSynchronize(c->panel_copy);
    for (auto e : c->chunk_h2d) cudaEventDestroy(e);
    for (auto e : c->chunk_ready) cudaEventDestroy(e);
    cudaEventDestroy(c->panel_ev);
    if (c->geom_ev) cudaEventDestroy(c->geom_ev);
    cudaStreamDestroy(c->panel_prep);
    cudaStreamDestroy(c->panel_copy);
  }
  for (auto* b : {&c->qh, &c->q1, &c->q0, &c->v, &c->v127, &c->skip}) b->release();
  for (auto* b : {&c->scale_d, &c->maxabs, &c->ystage, &c->rbar_in, &c->sum_d, &c->af, &c->var, &c->mu_d,
                  &c->invd_d, &c->cand_r, &c->cand_r_sorted, &c->cand_t, &c->cand_p, &c->full_r, &c->scratch_a,
                  &c->scratch_b, &c->scratch_c, &c->scratch_d, &c->pheno_sd, &c->cand_beta, &c->cand_se})
    b->release();
  for (auto* b : {&c->scale_f, &c->cq_f, &c->rbar, &c->mu_f, &c->invd_f}) b->release();
  for (auto* b : {&c->cq, &c->n_miss, &c->s_u, &c->ss_u}) b->release();
  c->gidx.release();
  c->keep_bits.release();
  c->max_abs_r.release();
  c->packed.release();
  c->raw_rows.release();
  c->flags.release();
  c->cand_key.release();
  c->cand_key_sorted.release();
  c->cand_rows.release();
  c->cand_cols.release();
  c->cand_count.release();
  c->counters.release();
  c->sort_tmp.release();
  c->new_row.release();
  c->full_out.release();
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  for (int i = 0; i < 2; ++i) {
    c->stage_buf[i].release();
    c->stage_raw[i].release();
    if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
    if (c->slot_free_ev[i]) cudaEventDestroy(c->slot_free_ev[i]);
    if (c->bgen_host[i]) cudaFreeHost(c->bgen_host[i]);
    if (c->h2d_ev[i]) cudaEventSynchronize(c->h2d_ev[i]);
    if (c->h2d_stage[i]) cudaFreeHost(c->h2d_stage[i]);
    if (c->h2d_ev[i]) cudaEventDestroy(c->h2d_ev[i]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return PG_OK;
}

int pg_ctx_stream(pg_ctx* c, void** stream) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(stream != nullptr, PG_ERR_INVALID, "null out");
  *stream = reinterpret_cast<void*>(c->stream);
  return PG_OK;
}

int pg_ctx_sync(pg_ctx* c) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_ctx_set_panel(pg_ctx* c, const double* ytil, int64_t n_kept, int64_t n_pheno, int64_t ld,
                     const int64_t* geno_row_index, int64_t n_samples_src) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(ytil != nullptr && geno_row_index != nullptr, PG_ERR_INVALID, "pg_ctx_set_panel: null input");
  PG_REQUIRE(ld >= n_pheno && n_pheno >= 1 && n_kept >= 1, PG_ERR_INVALID, "pg_ctx_set_panel: bad shape");
  PG_CHECK_STATUS(panel_drain(c));
  PG_CHECK_STATUS(c->ystage.ensure(static_cast<size_t>(n_kept) * n_pheno));
  if (ld == n_pheno) {
    PG_CUDA_CHECK(cudaMemcpyAsync(c->ystage.p, ytil, sizeof(double) * n_pheno * n_kept, cudaMemcpyHostToDevice,
                                  c->stream));
  } else {
    PG_CUDA_CHECK(cudaMemcpy2DAsync(c->ystage.p, sizeof(double) * n_pheno, ytil, sizeof(double) * ld,
                                    sizeof(double) * n_pheno, n_kept, cudaMemcpyHostToDevice, c->stream));
  }
  // the f64 staging buffer stays allocated: re-uploading a panel (e.g. per scan in a
  // service) must not pay a multi-GB cudaMalloc/cudaFree each time
  PG_CHECK_STATUS(upload_panel_common(c, c->ystage.p, n_kept, n_pheno, n_pheno, geno_row_index, n_samples_src));
  return PG_OK;
}

namespace {

// Host -> device copy of a large pageable buffer: 64 MB chunks are copied into two pinned
// bounce buffers by several host threads (one memcpy thread cannot feed the link) while
// the previous chunk's H2D runs on `s`. Already page-locked sources go straight through.
int upload_pageable(pg_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  constexpr size_t kChunk = kH2DBounce;
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost;
  cudaGetLastError();  // a pageable pointer may leave an error behind on older drivers
  if (pinned || bytes < 2 * kChunk) {
    PG_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return PG_OK;
  }
  for (int i = 0; i < 2; ++i) {
    if (c->h2d_stage[i] == nullptr) PG_CUDA_CHECK(cudaHostAlloc(&c->h2d_stage[i], kChunk, cudaHostAllocDefault));
    if (c->h2d_ev[i] == nullptr) PG_CUDA_CHECK(cudaEventCreateWithFlags(&c->h2d_ev[i], cudaEventDisableTiming));
  }
  const int nt = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  const char* from = static_cast<const char*>(src);
  char* to = static_cast<char*>(dst);
  int k = 0;
  for (size_t off = 0; off < bytes; off += kChunk, k ^= 1) {
    const size_t len = std::min(kChunk, bytes - off);
    PG_CUDA_CHECK(cudaEventSynchronize(c->h2d_ev[k]));  // this bounce buffer's previous H2D is done
    char* stage = static_cast<char*>(c->h2d_stage[k]);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
      th.emplace_back([=] {
        const size_t a = len * t / nt, b = len * (t + 1) / nt;
        std::memcpy(stage + a, from + off + a, b - a);
      });
    }
    for (auto& x : th) x.join();
    PG_CUDA_CHECK(cudaMemcpyAsync(to + off, stage, len, cudaMemcpyHostToDevice, s));
    PG_CUDA_CHECK(cudaEventRecord(c->h2d_ev[k], s));
  }
  return PG_OK;
}

}  // namespace

int pg_ctx_prepare_panel(pg_ctx* c, const double* y, int64_t n_kept, int64_t n_pheno, int64_t ld,
                         const double* basis_q, int64_t rank, uint8_t* zero_variance, double* sd) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(y != nullptr && zero_variance != nullptr && (rank == 0 || basis_q != nullptr), PG_ERR_INVALID,
             "pg_ctx_prepare_panel: null input");
  PG_REQUIRE(n_kept >= 1 && n_pheno >= 1 && ld >= n_pheno && rank >= 0, PG_ERR_INVALID,
             "pg_ctx_prepare_panel: bad shape");
  PG_CHECK_STATUS(panel_drain(c));
  cudaStream_t s = c->stream;
  PG_CHECK_STATUS(c->ystage.ensure(static_cast<size_t>(n_kept) * n_pheno));
  if (ld == n_pheno) {
    PG_CHECK_STATUS(upload_pageable(c, c->ystage.p, y, sizeof(double) * n_pheno * n_kept, s));
  } else {
    PG_CUDA_CHECK(cudaMemcpy2DAsync(c->ystage.p, sizeof(double) * n_pheno, y, sizeof(double) * ld,
                                    sizeof(double) * n_pheno, n_kept, cudaMemcpyHostToDevice, s));
  }
  if (rank > 0) {
    PG_CHECK_STATUS(c->prep_q.ensure(static_cast<size_t>(n_kept) * rank));
    PG_CUDA_CHECK(cudaMemcpyAsync(c->prep_q.p, basis_q, sizeof(double) * n_kept * rank, cudaMemcpyHostToDevice, s));
  }
  PG_CHECK_STATUS(c->prep_scratch.ensure(pg::panel_prep_scratch_doubles(n_kept, n_pheno, rank)));
  for (auto* b : {&c->prep_mean, &c->prep_centre, &c->prep_sd}) PG_CHECK_STATUS(b->ensure(n_pheno));
  PG_CHECK_STATUS(c->prep_flat.ensure(n_pheno));
  PG_CHECK_STATUS(c->prep_bad.ensure(1));
  pg::PanelPrepOut po;
  po.mean = c->prep_mean.p;
  po.centre = c->prep_centre.p;
  po.sd = c->prep_sd.p;
  po.flat = c->prep_flat.p;
  po.bad = c->prep_bad.p;
  PG_CHECK_STATUS(pg::panel_prepare(c->ystage.p, n_kept, n_pheno, rank ? c->prep_q.p : nullptr, rank,
                                    c->prep_scratch.p, po, s));
  int bad = 0;
  PG_CUDA_CHECK(cudaMemcpyAsync(&bad, c->prep_bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  PG_CUDA_CHECK(cudaMemcpyAsync(zero_variance, c->prep_flat.p, n_pheno, cudaMemcpyDeviceToHost, s));
  if (sd) PG_CUDA_CHECK(cudaMemcpyAsync(sd, c->prep_sd.p, sizeof(double) * n_pheno, cudaMemcpyDeviceToHost, s));
  PG_CUDA_CHECK(cudaStreamSynchronize(s));
  c->have_prepared = false;
  PG_REQUIRE(!bad, PG_ERR_INVALID, "standardize_columns requires finite input");
  c->have_prepared = true;
  c->prep_rows = n_kept;
  c->prep_cols = n_pheno;
  return PG_OK;
}

int pg_ctx_set_panel_async_cols(pg_ctx* c, const double* y, int64_t n_kept, int64_t n_pheno, int64_t ld,
                                int64_t col_begin, int64_t col_end, const double* basis_q, int64_t rank,
                                const int64_t* geno_row_index, int64_t n_samples_src, int64_t chunk_cols) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(y != nullptr && geno_row_index != nullptr && (rank == 0 || basis_q != nullptr), PG_ERR_INVALID,
             "pg_ctx_set_panel_async: null input");
  PG_REQUIRE(n_kept >= 1 && n_pheno >= 1 && rank >= 0 && chunk_cols >= 1 && col_begin >= 0 && col_end > col_begin &&
                 col_end <= n_pheno && ld >= col_end - col_begin,
             PG_ERR_INVALID, "pg_ctx_set_panel_async: bad shape");
  PG_REQUIRE(col_begin % kTileP == 0 && (col_end % kTileP == 0 || col_end == n_pheno), PG_ERR_INVALID,
             "pg_ctx_set_panel_async: a column range starts and ends on a multiple of %d phenotypes (or the last)",
             static_cast<int>(kTileP));
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, y) == cudaSuccess && attr.type == cudaMemoryTypeHost;
  cudaGetLastError();
  PG_REQUIRE(pinned, PG_ERR_INVALID,
             "pg_ctx_set_panel_async: the raw panel must be in page-locked host memory (else pg_ctx_prepare_panel)");
  PG_CHECK_STATUS(panel_drain(c));
  if (c->panel_prep == nullptr) {
    PG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->panel_copy, cudaStreamNonBlocking));
    PG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->panel_prep, cudaStreamNonBlocking));
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&c->panel_ev, cudaEventDisableTiming));
  }
  cudaStream_t ps = c->panel_prep, cs = c->panel_copy;
  // earlier scans on the compute stream may still read the current panel
  PG_CUDA_CHECK(cudaEventRecord(c->panel_ev, c->stream));
  PG_CUDA_CHECK(cudaStreamWaitEvent(ps, c->panel_ev, 0));
  PG_CUDA_CHECK(cudaStreamWaitEvent(cs, c->panel_ev, 0));
  PanelPlanes pp;
  PG_CHECK_STATUS(panel_geometry(c, n_kept, n_pheno, n_samples_src, geno_row_index, ps, pp));
  if (c->geom_ev == nullptr) PG_CUDA_CHECK(cudaEventCreateWithFlags(&c->geom_ev, cudaEventDisableTiming));
  PG_CUDA_CHECK(cudaEventRecord(c->geom_ev, ps));
  const int64_t chunk = round_up(std::max<int64_t>(chunk_cols, kTileP), kTileP);
  const int64_t n_ch = (col_end - col_begin + chunk - 1) / chunk;
  while (static_cast<int64_t>(c->chunk_ready.size()) < n_ch) {
    cudaEvent_t a, b;
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    c->chunk_h2d.push_back(a);
    c->chunk_ready.push_back(b);
  }
  c->chunk_pt.assign(n_ch + 1, 0);
  for (int64_t j = 0; j < n_ch; ++j) {
    const int64_t c0 = col_begin + j * chunk, c1 = std::min(col_end, c0 + chunk);
    c->chunk_pt[j] = c0 / kTileP;
    c->chunk_pt[j + 1] = c1 == n_pheno ? c->p_pad / kTileP : c1 / kTileP;
  }
  PG_CHECK_STATUS(c->ystage.ensure(static_cast<size_t>(n_kept) * (col_end - col_begin)));
  if (rank > 0) {
    PG_CHECK_STATUS(c->prep_q.ensure(static_cast<size_t>(n_kept) * rank));
    PG_CUDA_CHECK(cudaMemcpyAsync(c->prep_q.p, basis_q, sizeof(double) * n_kept * rank, cudaMemcpyHostToDevice, ps));
  }
  PG_CHECK_STATUS(
      c->prep_scratch.ensure(pg::panel_prep_scratch_doubles(n_kept, std::min(chunk, col_end - col_begin), rank)));
  for (auto* b : {&c->prep_mean, &c->prep_centre, &c->prep_sd}) PG_CHECK_STATUS(b->ensure(n_pheno));
  PG_CHECK_STATUS(c->prep_flat.ensure(n_pheno));
  PG_CHECK_STATUS(c->prep_bad.ensure(n_ch));
  PG_CHECK_STATUS(c->q0n.ensure(c->p_pad));
  c->prep_rows = n_kept;
  c->prep_cols = n_pheno;
  c->async_chunk = chunk;
  c->async_ld = ld;
  c->async_rank = rank;
  c->async_y = y;
  c->async_col0 = col_begin;
  c->async_col1 = col_end;
  c->chunk_issued = 0;
  c->n_chunks = n_ch;
  PG_CHECK_STATUS(panel_pump(c, 1));  // the first two chunks; the rest as they are needed
  c->panel_pending = true;
  c->async_flags = true;
  c->q0n_valid = true;
  c->have_prepared = false;
  c->have_panel = true;
  c->have_scan = false;
  c->have_basis = false;
  c->beta_on = false;
  return PG_OK;
}

int pg_ctx_set_panel_async(pg_ctx* c, const double* y, int64_t n_kept, int64_t n_pheno, int64_t ld,
                           const double* basis_q, int64_t rank, const int64_t* geno_row_index, int64_t n_samples_src,
                           int64_t chunk_cols) {
  PG_REQUIRE(ld >= n_pheno, PG_ERR_INVALID, "pg_ctx_set_panel_async: bad shape");
  return pg_ctx_set_panel_async_cols(c, y, n_kept, n_pheno, ld, 0, n_pheno, basis_q, rank, geno_row_index,
                                     n_samples_src, chunk_cols);
}

int pg_ctx_follow_panel(pg_ctx* f, pg_ctx* c) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(f != nullptr && f != c && f->device == c->device, PG_ERR_INVALID,
             "pg_ctx_follow_panel: need a second context on the same device");
  PG_REQUIRE(c->async_flags && c->leader == nullptr && c->follower == nullptr, PG_ERR_STATE,
             "pg_ctx_follow_panel: the source context has no pipelined panel of its own, or already a follower");
  PG_REQUIRE(f->f64_panel == c->f64_panel, PG_ERR_STATE,
             "pg_ctx_follow_panel: set the same precision (pg_ctx_set_f64_panel) on both contexts");
  PG_CHECK_STATUS(panel_drain(f));
  if (f->panel_prep == nullptr) {
    PG_CUDA_CHECK(cudaStreamCreateWithFlags(&f->panel_copy, cudaStreamNonBlocking));
    PG_CUDA_CHECK(cudaStreamCreateWithFlags(&f->panel_prep, cudaStreamNonBlocking));
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&f->panel_ev, cudaEventDisableTiming));
  }
  cudaStream_t fs = f->panel_prep;
  // the follower's earlier scans may still read its current panel
  PG_CUDA_CHECK(cudaEventRecord(f->panel_ev, f->stream));
  PG_CUDA_CHECK(cudaStreamWaitEvent(fs, f->panel_ev, 0));
  f->n_src = c->n_src;
  f->n_kept = c->n_kept;
  f->n_pheno = c->n_pheno;
  f->p_pad = c->p_pad;
  f->k_pad = c->k_pad;
  const size_t plane = static_cast<size_t>(c->p_pad) * c->k_pad;
  for (auto* b : {&f->qh, &f->q1, &f->q0}) PG_CHECK_STATUS(b->ensure(plane));
  PG_CHECK_STATUS(f->scale_d.ensure(c->p_pad));
  PG_CHECK_STATUS(f->scale_f.ensure(c->p_pad));
  PG_CHECK_STATUS(f->cq.ensure(c->p_pad));
  PG_CHECK_STATUS(f->cq_f.ensure(c->p_pad));
  PG_CHECK_STATUS(f->q0n.ensure(c->p_pad));
  if (c->f64_panel) {
    for (auto* b : {&f->qh_lo, &f->q1_lo, &f->q0_lo}) PG_CHECK_STATUS(b->ensure(plane));
    PG_CHECK_STATUS(f->cq_lo.ensure(c->p_pad));
  }
  const size_t kb_words = static_cast<size_t>(c->k_pad / 32 + 1);
  PG_CHECK_STATUS(f->gidx.ensure(c->n_kept));
  PG_CHECK_STATUS(f->keep_bits.ensure(kb_words));
  PG_CUDA_CHECK(cudaStreamWaitEvent(fs, c->geom_ev, 0));
  PG_CUDA_CHECK(cudaMemcpyAsync(f->gidx.p, c->gidx.p, sizeof(int64_t) * c->n_kept, cudaMemcpyDeviceToDevice, fs));
  PG_CUDA_CHECK(cudaMemcpyAsync(f->keep_bits.p, c->keep_bits.p, sizeof(uint32_t) * kb_words, cudaMemcpyDeviceToDevice, fs));
  while (f->chunk_ready.size() < c->chunk_ready.size()) {
    cudaEvent_t a, b;
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    PG_CUDA_CHECK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    f->chunk_h2d.push_back(a);
    f->chunk_ready.push_back(b);
  }
  f->n_chunks = c->n_chunks;
  f->chunk_pt = c->chunk_pt;
  {
    std::lock_guard<std::mutex> lock(c->pump_mu);
    for (int64_t j = 0; j < c->chunk_issued; ++j) PG_CHECK_STATUS(panel_copy_chunk(c, f, j));  // already issued
    c->follower = f;
    f->leader = c;
  }
  f->chunk_issued = 0;
  f->panel_pending = true;
  f->async_flags = false;
  f->q0n_valid = true;
  f->have_prepared = false;
  f->have_panel = true;
  f->have_scan = false;
  f->have_basis = false;
  f->beta_on = false;
  return PG_OK;
}

int pg_ctx_panel_async_wait(pg_ctx* c, uint8_t* zero_variance, double* sd) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->async_flags, PG_ERR_STATE, "pg_ctx_panel_async_wait: no pipelined panel (pg_ctx_set_panel_async)");
  PG_CHECK_STATUS(panel_pump(c, c->n_chunks - 1));
  cudaStream_t ps = c->panel_prep;
  std::vector<int> bad(static_cast<size_t>(c->n_chunks), 0);
  PG_CUDA_CHECK(cudaMemcpyAsync(bad.data(), c->prep_bad.p, sizeof(int) * c->n_chunks, cudaMemcpyDeviceToHost, ps));
  const int64_t c0 = c->async_col0, nc = c->async_col1 - c->async_col0;  // the prepared columns
  if (zero_variance)
    PG_CUDA_CHECK(cudaMemcpyAsync(zero_variance, c->prep_flat.p + c0, nc, cudaMemcpyDeviceToHost, ps));
  if (sd) PG_CUDA_CHECK(cudaMemcpyAsync(sd, c->prep_sd.p + c0, sizeof(double) * nc, cudaMemcpyDeviceToHost, ps));
  PG_CUDA_CHECK(cudaStreamSynchronize(ps));
  c->panel_pending = false;  // every chunk is complete: no stream needs to wait any more
  for (int v : bad) PG_REQUIRE(!v, PG_ERR_INVALID, "standardize_columns requires finite input");
  return PG_OK;
}

int pg_ctx_fetch_prepared_panel(pg_ctx* c, double* out) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_prepared, PG_ERR_STATE, "no prepared panel (pg_ctx_prepare_panel)");
  PG_REQUIRE(out != nullptr, PG_ERR_INVALID, "null output");
  PG_CUDA_CHECK(cudaMemcpyAsync(out, c->ystage.p, sizeof(double) * c->prep_rows * c->prep_cols,
                                cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_ctx_commit_panel(pg_ctx* c, const int64_t* kept_cols, int64_t n_cols, const int64_t* geno_row_index,
                        int64_t n_samples_src) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_prepared, PG_ERR_STATE, "pg_ctx_commit_panel: no prepared panel (pg_ctx_prepare_panel)");
  PG_REQUIRE(kept_cols != nullptr && geno_row_index != nullptr && n_cols >= 1, PG_ERR_INVALID,
             "pg_ctx_commit_panel: null input or no columns");
  for (int64_t i = 0; i < n_cols; ++i)
    PG_REQUIRE(kept_cols[i] >= 0 && kept_cols[i] < c->prep_cols, PG_ERR_INVALID,
               "pg_ctx_commit_panel: column %lld out of range", (long long)kept_cols[i]);
  PG_CHECK_STATUS(c->colmap.ensure(n_cols));
  PG_CUDA_CHECK(
      cudaMemcpyAsync(c->colmap.p, kept_cols, sizeof(int64_t) * n_cols, cudaMemcpyHostToDevice, c->stream));
  return upload_panel_common(c, c->ystage.p, c->prep_rows, n_cols, c->prep_cols, geno_row_index, n_samples_src,
                             c->colmap.p);
}

int pg_ctx_set_panel_device(pg_ctx* c, const double* d_ytil, int64_t n_kept, int64_t n_pheno, int64_t ld,
                            const int64_t* geno_row_index, int64_t n_samples_src) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(d_ytil != nullptr && geno_row_index != nullptr, PG_ERR_INVALID, "pg_ctx_set_panel_device: null input");
  return upload_panel_common(c, d_ytil, n_kept, n_pheno, ld, geno_row_index, n_samples_src);
}

int pg_ctx_panel_bytes(pg_ctx* c, int64_t* bytes) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "no panel");
  *bytes = 3 * c->p_pad * c->k_pad + c->p_pad * (8 + 4 + 8 + 4);
  if (c->f64_panel) *bytes += 3 * c->p_pad * c->k_pad + c->p_pad * 8;  // the lo level
  return PG_OK;
}

int pg_ctx_export_panel(pg_ctx* c, void* d_dst) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "no panel");
  PG_CHECK_STATUS(panel_wait_all(c, c->stream));
  uint8_t* d = static_cast<uint8_t*>(d_dst);
  const size_t plane = static_cast<size_t>(c->p_pad) * c->k_pad;
  const size_t pp = static_cast<size_t>(c->p_pad);
  PG_CUDA_CHECK(cudaMemcpyAsync(d, c->qh.p, plane, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(d + plane, c->q1.p, plane, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(d + 2 * plane, c->q0.p, plane, cudaMemcpyDeviceToDevice, c->stream));
  uint8_t* tail = d + 3 * plane;
  PG_CUDA_CHECK(cudaMemcpyAsync(tail, c->scale_d.p, 8 * pp, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(tail + 8 * pp, c->scale_f.p, 4 * pp, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(tail + 12 * pp, c->cq.p, 8 * pp, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(tail + 20 * pp, c->cq_f.p, 4 * pp, cudaMemcpyDeviceToDevice, c->stream));
  if (c->f64_panel) {
    uint8_t* lo = tail + 24 * pp;
    PG_CUDA_CHECK(cudaMemcpyAsync(lo, c->qh_lo.p, plane, cudaMemcpyDeviceToDevice, c->stream));
    PG_CUDA_CHECK(cudaMemcpyAsync(lo + plane, c->q1_lo.p, plane, cudaMemcpyDeviceToDevice, c->stream));
    PG_CUDA_CHECK(cudaMemcpyAsync(lo + 2 * plane, c->q0_lo.p, plane, cudaMemcpyDeviceToDevice, c->stream));
    PG_CUDA_CHECK(cudaMemcpyAsync(lo + 3 * plane, c->cq_lo.p, 8 * pp, cudaMemcpyDeviceToDevice, c->stream));
  }
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

// Panel rows [row_begin, row_end) as one device buffer: the three limb planes' rows, then
// scale_d (f64), scale_f (f32), Cq (i64), Cq_f (f32), ||q0|| (f32) per row, then the lo level
// (three planes + Cq_lo) in F64 mode. Multi-GPU: each rank prepares its share of the
// phenotypes and the shares are all-gathered (bench.py, distributed panel preparation).
static int64_t panel_rows_bytes(const pg_ctx* c, int64_t r) {
  int64_t b = 3 * r * c->k_pad + r * (8 + 4 + 8 + 4 + 4);
  if (c->f64_panel) b += 3 * r * c->k_pad + r * 8;
  return b;
}

static int panel_rows_copy(pg_ctx* c, uint8_t* buf, int64_t row_begin, int64_t row_end, bool to_buf) {
  const int64_t r = row_end - row_begin;
  const size_t plane = static_cast<size_t>(r) * c->k_pad, off = static_cast<size_t>(row_begin) * c->k_pad;
  cudaStream_t s = c->stream;
  auto cp = [&](void* panel, size_t bytes, uint8_t*& cursor) -> int {
    if (to_buf)
      PG_CUDA_CHECK(cudaMemcpyAsync(cursor, panel, bytes, cudaMemcpyDeviceToDevice, s));
    else
      PG_CUDA_CHECK(cudaMemcpyAsync(panel, cursor, bytes, cudaMemcpyDeviceToDevice, s));
    cursor += bytes;
    return PG_OK;
  };
  uint8_t* cur = buf;
  PG_CHECK_STATUS(cp(c->qh.p + off, plane, cur));
  PG_CHECK_STATUS(cp(c->q1.p + off, plane, cur));
  PG_CHECK_STATUS(cp(c->q0.p + off, plane, cur));
  PG_CHECK_STATUS(cp(c->scale_d.p + row_begin, 8 * r, cur));
  PG_CHECK_STATUS(cp(c->scale_f.p + row_begin, 4 * r, cur));
  PG_CHECK_STATUS(cp(c->cq.p + row_begin, 8 * r, cur));
  PG_CHECK_STATUS(cp(c->cq_f.p + row_begin, 4 * r, cur));
  PG_CHECK_STATUS(cp(c->q0n.p + row_begin, 4 * r, cur));
  if (c->f64_panel) {
    PG_CHECK_STATUS(cp(c->qh_lo.p + off, plane, cur));
    PG_CHECK_STATUS(cp(c->q1_lo.p + off, plane, cur));
    PG_CHECK_STATUS(cp(c->q0_lo.p + off, plane, cur));
    PG_CHECK_STATUS(cp(c->cq_lo.p + row_begin, 8 * r, cur));
  }
  PG_CUDA_CHECK(cudaStreamSynchronize(s));
  return PG_OK;
}

int pg_ctx_panel_rows_bytes(pg_ctx* c, int64_t n_rows, int64_t* bytes) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel && bytes != nullptr && n_rows >= 0, PG_ERR_STATE, "pg_ctx_panel_rows_bytes: no panel");
  *bytes = panel_rows_bytes(c, n_rows);
  return PG_OK;
}

int pg_ctx_export_panel_rows(pg_ctx* c, void* d_dst, int64_t row_begin, int64_t row_end) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel && c->q0n_valid, PG_ERR_STATE, "pg_ctx_export_panel_rows: no (pipelined) panel");
  PG_REQUIRE(d_dst != nullptr && row_begin >= 0 && row_end > row_begin && row_end <= c->p_pad, PG_ERR_INVALID,
             "pg_ctx_export_panel_rows: bad row range");
  PG_CHECK_STATUS(panel_wait_all(c, c->stream));
  return panel_rows_copy(c, static_cast<uint8_t*>(d_dst), row_begin, row_end, true);
}

int pg_ctx_import_panel_rows(pg_ctx* c, const void* d_src, int64_t row_begin, int64_t row_end) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel && c->q0n_valid, PG_ERR_STATE,
             "pg_ctx_import_panel_rows: set the panel geometry first (pg_ctx_set_panel_async_cols)");
  PG_REQUIRE(d_src != nullptr && row_begin >= 0 && row_end > row_begin && row_end <= c->p_pad, PG_ERR_INVALID,
             "pg_ctx_import_panel_rows: bad row range");
  PG_CHECK_STATUS(panel_wait_all(c, c->stream));
  return panel_rows_copy(c, const_cast<uint8_t*>(static_cast<const uint8_t*>(d_src)), row_begin, row_end, false);
}

int pg_ctx_clone_panel(pg_ctx* dst, pg_ctx* src) {
  PG_CHECK_STATUS(ctx_check(src));
  PG_REQUIRE(dst != nullptr && dst != src, PG_ERR_INVALID, "pg_ctx_clone_panel: need two distinct contexts");
  PG_REQUIRE(src->have_panel, PG_ERR_STATE, "pg_ctx_clone_panel: the source context has no panel");
  PG_REQUIRE(dst->device == src->device, PG_ERR_INVALID, "pg_ctx_clone_panel: contexts on different devices");
  PG_REQUIRE(dst->f64_panel == src->f64_panel, PG_ERR_STATE,
             "pg_ctx_clone_panel: set the same precision (pg_ctx_set_f64_panel) on both contexts");
  int64_t bytes = 0;
  PG_CHECK_STATUS(pg_ctx_panel_bytes(src, &bytes));
  std::vector<int64_t> gidx(static_cast<size_t>(src->n_kept));
  void* tmp = nullptr;
  PG_CUDA_CHECK(cudaMalloc(&tmp, static_cast<size_t>(bytes)));
  int rc = pg_ctx_export_panel(src, tmp);  // waits for a pipelined preparation; synchronous
  if (rc == PG_OK) {
    const cudaError_t e = cudaMemcpy(gidx.data(), src->gidx.p, sizeof(int64_t) * gidx.size(), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      pg::set_error("pg_ctx_clone_panel: %s", cudaGetErrorString(e));
      rc = PG_ERR_CUDA;
    }
  }
  if (rc == PG_OK) rc = pg_ctx_import_panel(dst, tmp, src->n_kept, src->n_pheno, gidx.data(), src->n_src);
  cudaFree(tmp);
  return rc;
}

int pg_ctx_import_panel(pg_ctx* c, const void* d_src, int64_t n_kept, int64_t n_pheno,
                        const int64_t* geno_row_index, int64_t n_samples_src) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(d_src != nullptr && geno_row_index != nullptr, PG_ERR_INVALID, "pg_ctx_import_panel: null input");
  PG_CHECK_STATUS(panel_drain(c));
  // geometry + keep mask exactly as set_panel would build them
  std::vector<uint32_t> bits;
  c->n_src = n_samples_src;
  c->n_kept = n_kept;
  c->n_pheno = n_pheno;
  c->p_pad = round_up(n_pheno, kTileP);
  PG_REQUIRE(round_up(n_samples_src, 64) <= (int64_t(1) << 30), PG_ERR_CONFIG, "%lld genotype samples: too many",
             (long long)n_samples_src);
  c->k_pad = round_up(n_samples_src, 64);
  bits.assign(c->k_pad / 32 + 1, 0u);
  for (int64_t i = 0; i < n_kept; ++i) {
    const int64_t g = geno_row_index[i];
    PG_REQUIRE(g >= 0 && g < n_samples_src, PG_ERR_INVALID, "geno_row_index out of range");
    bits[g >> 5] |= 1u << (g & 31);
  }
  const size_t plane = static_cast<size_t>(c->p_pad) * c->k_pad;
  const size_t pp = static_cast<size_t>(c->p_pad);
  PG_CHECK_STATUS(c->qh.ensure(plane));
  PG_CHECK_STATUS(c->q1.ensure(plane));
  PG_CHECK_STATUS(c->q0.ensure(plane));
  PG_CHECK_STATUS(c->scale_d.ensure(pp));
  PG_CHECK_STATUS(c->scale_f.ensure(pp));
  PG_CHECK_STATUS(c->cq.ensure(pp));
  PG_CHECK_STATUS(c->cq_f.ensure(pp));
  PG_CHECK_STATUS(c->gidx.ensure(n_kept));
  PG_CHECK_STATUS(c->keep_bits.ensure(bits.size()));
  const uint8_t* s = static_cast<const uint8_t*>(d_src);
  c->q0n_valid = false;
  PG_CUDA_CHECK(cudaMemcpyAsync(c->qh.p, s, plane, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->q1.p, s + plane, plane, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->q0.p, s + 2 * plane, plane, cudaMemcpyDeviceToDevice, c->stream));
  const uint8_t* tail = s + 3 * plane;
  PG_CUDA_CHECK(cudaMemcpyAsync(c->scale_d.p, tail, 8 * pp, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->scale_f.p, tail + 8 * pp, 4 * pp, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->cq.p, tail + 12 * pp, 8 * pp, cudaMemcpyDeviceToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->cq_f.p, tail + 20 * pp, 4 * pp, cudaMemcpyDeviceToDevice, c->stream));
  if (c->f64_panel) {
    PG_CHECK_STATUS(c->qh_lo.ensure(plane));
    PG_CHECK_STATUS(c->q1_lo.ensure(plane));
    PG_CHECK_STATUS(c->q0_lo.ensure(plane));
    PG_CHECK_STATUS(c->cq_lo.ensure(pp));
    const uint8_t* lo = tail + 24 * pp;
    PG_CUDA_CHECK(cudaMemcpyAsync(c->qh_lo.p, lo, plane, cudaMemcpyDeviceToDevice, c->stream));
    PG_CUDA_CHECK(cudaMemcpyAsync(c->q1_lo.p, lo + plane, plane, cudaMemcpyDeviceToDevice, c->stream));
    PG_CUDA_CHECK(cudaMemcpyAsync(c->q0_lo.p, lo + 2 * plane, plane, cudaMemcpyDeviceToDevice, c->stream));
    PG_CUDA_CHECK(cudaMemcpyAsync(c->cq_lo.p, lo + 3 * plane, 8 * pp, cudaMemcpyDeviceToDevice, c->stream));
  }
  PG_CUDA_CHECK(cudaMemcpyAsync(c->gidx.p, geno_row_index, sizeof(int64_t) * n_kept, cudaMemcpyHostToDevice,
                                c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->keep_bits.p, bits.data(), sizeof(uint32_t) * bits.size(), cudaMemcpyHostToDevice,
                                c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->have_panel = true;
  c->have_scan = false;
  c->have_basis = false;
  c->beta_on = false;  // phenotype scales belong to the previous panel's columns
  return PG_OK;
}

int pg_ctx_set_scan(pg_ctx* c, double df, int mode, const double* r_bar) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_ctx_set_scan: no panel");
  PG_REQUIRE(df >= 1.0, PG_ERR_INVALID, "degrees of freedom %g < 1", df);
  PG_REQUIRE(mode == PG_MODE_THRESHOLD || mode == PG_MODE_TOPK || mode == PG_MODE_FULL, PG_ERR_INVALID,
             "unknown output mode %d", mode);
  PG_REQUIRE(mode == PG_MODE_FULL || r_bar != nullptr, PG_ERR_INVALID, "r_bar required for THRESHOLD/TOPK");
  c->df = df;
  c->mode = mode;
  c->track_max_abs_r = false;
  PG_CHECK_STATUS(c->rbar.ensure(c->p_pad));
  PG_CHECK_STATUS(c->rbar_in.ensure(c->n_pheno));
  PG_CHECK_STATUS(c->max_abs_r.ensure(c->p_pad));
  PG_CUDA_CHECK(cudaMemsetAsync(c->max_abs_r.p, 0, sizeof(unsigned long long) * c->p_pad, c->stream));
  if (r_bar != nullptr) {
    PG_CUDA_CHECK(
        cudaMemcpyAsync(c->rbar_in.p, r_bar, sizeof(double) * c->n_pheno, cudaMemcpyHostToDevice, c->stream));
    rbar_kernel<<<static_cast<unsigned>((c->p_pad + 255) / 256), 256, 0, c->stream>>>(c->rbar_in.p, c->n_pheno,
                                                                                       c->p_pad, c->rbar.p);
    PG_CUDA_CHECK(cudaGetLastError());
  }
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->have_scan = true;
  return PG_OK;
}

int pg_ctx_set_basis(pg_ctx* c, const double* q, int64_t n_kept, int64_t rank) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_ctx_set_basis: set the panel first");
  PG_CHECK_STATUS(panel_wait_all(c, c->stream));
  if (q == nullptr || rank <= 1) {
    c->have_basis = false;
    return PG_OK;
  }
  PG_REQUIRE(n_kept == c->n_kept, PG_ERR_INVALID, "pg_ctx_set_basis: %lld rows, panel has %lld kept samples",
             (long long)n_kept, (long long)c->n_kept);
  PG_REQUIRE(rank - 1 <= kTileP, PG_ERR_INVALID, "pg_ctx_set_basis: rank %lld > %d", (long long)rank, kTileP + 1);
  const size_t plane = static_cast<size_t>(kTileP) * c->k_pad;
  PG_CHECK_STATUS(c->bq_h.ensure(plane));
  PG_CHECK_STATUS(c->bq_1.ensure(plane));
  PG_CHECK_STATUS(c->bq_0.ensure(plane));
  PG_CHECK_STATUS(c->bscale_d.ensure(kTileP));
  PG_CHECK_STATUS(c->bscale_f.ensure(kTileP));
  PG_CHECK_STATUS(c->bcq.ensure(kTileP));
  PG_CHECK_STATUS(c->bcq_f.ensure(kTileP));
  PG_CHECK_STATUS(c->bmaxabs.ensure(kTileP));
  PG_CHECK_STATUS(c->bstage.ensure(static_cast<size_t>(n_kept) * rank));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->bstage.p, q, sizeof(double) * n_kept * rank, cudaMemcpyHostToDevice, c->stream));
  PanelPlanes pp;
  pp.qh = c->bq_h.p;
  pp.q1 = c->bq_1.p;
  pp.q0 = c->bq_0.p;
  pp.scale_d = c->bscale_d.p;
  pp.scale_f = c->bscale_f.p;
  pp.cq = c->bcq.p;
  pp.cq_f = c->bcq_f.p;
  // columns 1..rank-1 (the intercept column contributes exactly 0 after centring)
  PG_CHECK_STATUS(panel_quantize(c->bstage.p + 1, n_kept, rank - 1, rank, nullptr, c->gidx.p, c->k_pad, kTileP, pp,
                                 c->bmaxabs.p, c->stream));
  // w_j = sum over ALL kept samples: no centring term (Cq = 0 in the epilogue formula)
  PG_CUDA_CHECK(cudaMemsetAsync(c->bcq.p, 0, sizeof(long long) * kTileP, c->stream));
  PG_CUDA_CHECK(cudaMemsetAsync(c->bcq_f.p, 0, sizeof(float) * kTileP, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->bstage.release();
  c->basis_cols = rank - 1;
  c->have_basis = true;
  return PG_OK;
}

int pg_ctx_set_beta_scale(pg_ctx* c, const double* pheno_sd, int64_t n_pheno) {
  PG_CHECK_STATUS(ctx_check(c));
  if (pheno_sd == nullptr) {
    c->beta_on = false;
    return PG_OK;
  }
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_ctx_set_beta_scale: no panel");
  PG_REQUIRE(n_pheno == c->n_pheno, PG_ERR_INVALID, "pg_ctx_set_beta_scale: %lld scales for %lld phenotypes",
             (long long)n_pheno, (long long)c->n_pheno);
  for (int64_t j = 0; j < n_pheno; ++j)
    PG_REQUIRE(std::isfinite(pheno_sd[j]) && pheno_sd[j] > 0.0, PG_ERR_INVALID,
               "pg_ctx_set_beta_scale: phenotype %lld has sd %g", (long long)j, pheno_sd[j]);
  PG_CHECK_STATUS(c->pheno_sd.ensure(c->p_pad));
  PG_CUDA_CHECK(cudaMemsetAsync(c->pheno_sd.p, 0, sizeof(double) * c->p_pad, c->stream));
  PG_CUDA_CHECK(
      cudaMemcpyAsync(c->pheno_sd.p, pheno_sd, sizeof(double) * n_pheno, cudaMemcpyHostToDevice, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->beta_on = true;
  return PG_OK;
}

int pg_ctx_debug_candidate_base(pg_ctx* c, uint64_t base) {
  PG_CHECK_STATUS(ctx_check(c));
  c->cand_base = base;
  return PG_OK;
}

int pg_ctx_set_wide_digits(pg_ctx* c, int enable) {
  PG_CHECK_STATUS(ctx_check(c));
  c->wide_digits = enable != 0;
  return PG_OK;
}

int pg_ctx_set_two_limb_premask(pg_ctx* c, int enable) {
  PG_CHECK_STATUS(ctx_check(c));
  c->two_limb = enable != 0;
  return PG_OK;
}

int pg_ctx_set_f64_panel(pg_ctx* c, int enable) {
  PG_CHECK_STATUS(ctx_check(c));
  if ((enable != 0) != c->f64_panel) {
    c->f64_panel = enable != 0;
    c->have_panel = false;  // the panel's levels change: upload it (again) after this call
    c->have_scan = false;
  }
  return PG_OK;
}

int pg_ctx_set_missing_side_gemm(pg_ctx* c, int enable) {
  PG_CHECK_STATUS(ctx_check(c));
  c->side_missing = enable != 0;
  return PG_OK;
}

int pg_ctx_set_fused_decode(pg_ctx* c, int enable) {
  PG_CHECK_STATUS(ctx_check(c));
  c->fused_decode = enable != 0;
  return PG_OK;
}

int pg_ctx_set_rbar(pg_ctx* c, const double* r_bar) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_scan && r_bar != nullptr, PG_ERR_STATE, "pg_ctx_set_rbar: scan not configured");
  PG_CUDA_CHECK(cudaMemcpyAsync(c->rbar_in.p, r_bar, sizeof(double) * c->n_pheno, cudaMemcpyHostToDevice, c->stream));
  rbar_kernel<<<static_cast<unsigned>((c->p_pad + 255) / 256), 256, 0, c->stream>>>(c->rbar_in.p, c->n_pheno, c->p_pad,
                                                                                     c->rbar.p);
  PG_CUDA_CHECK(cudaGetLastError());
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_scan(pg_ctx* c, int kind, const void* data, int64_t n_markers, int64_t row_bytes, pg_batch_info* info) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_scan: no panel uploaded (pg_ctx_set_panel)");
  const int64_t expect = expected_row_bytes(kind, c->n_src);
  PG_REQUIRE(expect > 0, PG_ERR_INVALID, "unknown genotype kind %d", kind);
  PG_REQUIRE(row_bytes == expect, PG_ERR_FORMAT, "packed row has %lld bytes, expected %lld for %lld samples",
             (long long)row_bytes, (long long)expect, (long long)c->n_src);
  PG_REQUIRE(data != nullptr && n_markers >= 1, PG_ERR_INVALID, "pg_scan: empty batch");
  const int64_t pitch = round_up(row_bytes, 16);
  PG_CHECK_STATUS(c->packed.ensure(static_cast<size_t>(pitch) * n_markers));
  PG_CHECK_STATUS(upload_rows(data, n_markers, row_bytes, pitch, c->raw_rows, c->packed.p, c->stream));
  return scan_common(c, kind, c->packed.p, n_markers, pitch, info);
}

int pg_stage(pg_ctx* c, int slot, int kind, const void* data, int64_t n_markers, int64_t row_bytes) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(slot == 0 || slot == 1, PG_ERR_INVALID, "pg_stage: slot must be 0 or 1");
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_stage: no panel uploaded (pg_ctx_set_panel)");
  const int64_t expect = expected_row_bytes(kind, c->n_src);
  PG_REQUIRE(expect > 0, PG_ERR_INVALID, "unknown genotype kind %d", kind);
  PG_REQUIRE(row_bytes == expect, PG_ERR_FORMAT, "packed row has %lld bytes, expected %lld for %lld samples",
             (long long)row_bytes, (long long)expect, (long long)c->n_src);
  PG_REQUIRE(data != nullptr && n_markers >= 1, PG_ERR_INVALID, "pg_stage: empty batch");
  const int64_t pitch = round_up(row_bytes, 16);
  // the slot may still be read by the scan that last used it
  PG_CUDA_CHECK(cudaStreamWaitEvent(c->copy_stream, c->slot_free_ev[slot], 0));
  if (c->stage_buf[slot].cap < static_cast<size_t>(pitch) * n_markers) {
    PG_CUDA_CHECK(cudaStreamSynchronize(c->copy_stream));
    PG_CHECK_STATUS(c->stage_buf[slot].ensure(static_cast<size_t>(pitch) * n_markers));
  }
  if (c->stage_raw[slot].cap < static_cast<size_t>(row_bytes) * n_markers) {
    PG_CUDA_CHECK(cudaStreamSynchronize(c->copy_stream));
    PG_CHECK_STATUS(c->stage_raw[slot].ensure(static_cast<size_t>(row_bytes) * n_markers));
  }
  PG_CHECK_STATUS(upload_rows(data, n_markers, row_bytes, pitch, c->stage_raw[slot], c->stage_buf[slot].p,
                              c->copy_stream));
  PG_CUDA_CHECK(cudaEventRecord(c->stage_ev[slot], c->copy_stream));
  c->stage_kind[slot] = kind;
  c->stage_data[slot] = c->stage_buf[slot].p;
  c->stage_probs_off[slot] = 0;
  c->stage_ploidy_off[slot] = -1;
  c->stage_m[slot] = n_markers;
  c->stage_pitch[slot] = pitch;
  return PG_OK;
}

int pg_stage_bgen_begin(pg_ctx* c, int slot, const void* blob, int64_t blob_bytes, const int64_t* block_off,
                        const int64_t* block_size, int64_t count) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(slot == 0 || slot == 1, PG_ERR_INVALID, "pg_stage_bgen: slot must be 0 or 1");
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_stage_bgen: no panel uploaded (pg_ctx_set_panel)");
  PG_REQUIRE(blob != nullptr && block_off != nullptr && block_size != nullptr && count >= 1, PG_ERR_INVALID,
             "pg_stage_bgen: empty batch or null argument");
  PG_REQUIRE(c->bgen_pending[slot] == 0, PG_ERR_STATE, "pg_stage_bgen: slot %d already has a batch in flight", slot);
  for (int64_t i = 0; i < count; ++i)
    PG_REQUIRE(block_off[i] >= 0 && block_size[i] >= 0 && block_off[i] + block_size[i] <= blob_bytes,
               PG_ERR_INVALID, "pg_stage_bgen: block %lld outside the blob", (long long)i);
  const int64_t n = c->n_src;
  const int64_t raw_stride = round_up(10 + 5 * n, 16);
  cudaStream_t cs = c->copy_stream;
  // the slot's buffers may still be read by the scan that last used it
  PG_CUDA_CHECK(cudaStreamWaitEvent(cs, c->slot_free_ev[slot], 0));
  if (c->bgen_blob[slot].cap < static_cast<size_t>(blob_bytes + 16) ||
      c->bgen_raw[slot].cap < static_cast<size_t>(raw_stride) * count || c->bgen_off[slot].cap < static_cast<size_t>(count) ||
      c->bgen_tok[slot].cap < static_cast<size_t>(pg::inflate_token_stride(raw_stride)) * count ||
      c->bgen_ntok[slot].cap < static_cast<size_t>(2 * count))
    PG_CUDA_CHECK(cudaStreamSynchronize(cs));  // reallocation below must not free memory in use
  PG_CHECK_STATUS(c->bgen_blob[slot].ensure(blob_bytes + 16));  // the decoder reads ahead <= 8 B past a stream
  PG_CHECK_STATUS(c->bgen_raw[slot].ensure(static_cast<size_t>(raw_stride) * count));
  for (auto* b : {&c->bgen_off[slot], &c->bgen_size[slot], &c->bgen_len[slot]}) PG_CHECK_STATUS(b->ensure(count));
  PG_CHECK_STATUS(c->bgen_zstatus[slot].ensure(count));
  PG_CHECK_STATUS(c->bgen_bits[slot].ensure(count));
  PG_CHECK_STATUS(c->bgen_tok[slot].ensure(static_cast<size_t>(pg::inflate_token_stride(raw_stride)) * count));
  PG_CHECK_STATUS(c->bgen_ntok[slot].ensure(2 * count));
  PG_CHECK_STATUS(c->bgen_diag[slot].ensure(3 * count));
  PG_CHECK_STATUS(c->bgen_summary[slot].ensure(2));
  if (c->bgen_host[slot] == nullptr) PG_CUDA_CHECK(cudaHostAlloc(&c->bgen_host[slot], 64, cudaHostAllocDefault));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->bgen_blob[slot].p, blob, blob_bytes, cudaMemcpyHostToDevice, cs));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->bgen_off[slot].p, block_off, sizeof(int64_t) * count, cudaMemcpyHostToDevice, cs));
  PG_CUDA_CHECK(
      cudaMemcpyAsync(c->bgen_size[slot].p, block_size, sizeof(int64_t) * count, cudaMemcpyHostToDevice, cs));
  // genotype block = u32 uncompressed length + zlib stream
  PG_CHECK_STATUS(pg::inflate_streams(c->bgen_blob[slot].p, c->bgen_off[slot].p, c->bgen_size[slot].p, count, 4,
                                      c->bgen_raw[slot].p, raw_stride, c->bgen_len[slot].p, c->bgen_zstatus[slot].p,
                                      cs, c->bgen_tok[slot].p, c->bgen_ntok[slot].p));
  PG_CUDA_CHECK(cudaMemsetAsync(c->bgen_summary[slot].p, 0xFF, sizeof(unsigned long long), cs));
  PG_CUDA_CHECK(cudaMemsetAsync(c->bgen_summary[slot].p + 1, 0, sizeof(unsigned long long), cs));
  PG_CHECK_STATUS(pg::bgen_validate(c->bgen_blob[slot].p, c->bgen_off[slot].p, c->bgen_size[slot].p,
                                    c->bgen_raw[slot].p, raw_stride, c->bgen_len[slot].p, c->bgen_zstatus[slot].p,
                                    count, n, c->bgen_diag[slot].p, c->bgen_bits[slot].p, c->bgen_summary[slot].p,
                                    cs));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->bgen_host[slot], c->bgen_summary[slot].p, 2 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, cs));
  PG_CUDA_CHECK(cudaEventRecord(c->stage_ev[slot], cs));
  c->bgen_pending[slot] = count;
  return PG_OK;
}

int pg_stage_bgen_end(pg_ctx* c, int slot, int64_t* diag) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(slot == 0 || slot == 1, PG_ERR_INVALID, "pg_stage_bgen_end: slot must be 0 or 1");
  PG_REQUIRE(diag != nullptr, PG_ERR_INVALID, "pg_stage_bgen_end: null diag");
  const int64_t count = c->bgen_pending[slot];
  PG_REQUIRE(count > 0, PG_ERR_STATE, "pg_stage_bgen_end: no batch in flight in slot %d", slot);
  c->bgen_pending[slot] = 0;
  diag[0] = diag[1] = diag[2] = diag[3] = 0;
  PG_CUDA_CHECK(cudaEventSynchronize(c->stage_ev[slot]));
  const unsigned long long* summary = static_cast<const unsigned long long*>(c->bgen_host[slot]);
  if (summary[0] != ~0ull) {
    long long d3[3] = {0, 0, 0};
    PG_CUDA_CHECK(cudaMemcpy(d3, c->bgen_diag[slot].p + 3 * summary[0], sizeof(d3), cudaMemcpyDeviceToHost));
    diag[0] = static_cast<int64_t>(summary[0]);
    diag[1] = d3[0];
    diag[2] = d3[1];
    diag[3] = d3[2];
    pg::set_error("BGEN block %lld failed validation (reason %lld)", (long long)summary[0], d3[0]);
    return PG_ERR_FORMAT;
  }
  const int64_t n = c->n_src;
  const int64_t raw_stride = round_up(10 + 5 * n, 16);
  const bool wide16 = (summary[1] & 2ull) != 0;
  const int64_t row_bytes = wide16 ? 5 * n : 3 * n;
  const int64_t pitch = round_up(row_bytes, 16);
  c->stage_kind[slot] = wide16 ? PG_GENO_BGEN16 : PG_GENO_BGEN8;
  c->stage_m[slot] = count;
  if (!wide16) {
    // all-8-bit batch: the decoders read the inflated blocks in place (no repack pass)
    c->stage_data[slot] = c->bgen_raw[slot].p;
    c->stage_pitch[slot] = raw_stride;
    c->stage_probs_off[slot] = 10 + n;
    c->stage_ploidy_off[slot] = 8;
    return PG_OK;
  }
  cudaStream_t cs = c->copy_stream;
  if (c->stage_buf[slot].cap < static_cast<size_t>(pitch) * count) {
    PG_CUDA_CHECK(cudaStreamSynchronize(cs));
    PG_CHECK_STATUS(c->stage_buf[slot].ensure(static_cast<size_t>(pitch) * count));
  }
  PG_CHECK_STATUS(pg::bgen_repack(c->bgen_raw[slot].p, raw_stride, c->bgen_bits[slot].p, count, n, wide16,
                                  c->stage_buf[slot].p, pitch, cs));
  PG_CUDA_CHECK(cudaEventRecord(c->stage_ev[slot], cs));
  c->stage_data[slot] = c->stage_buf[slot].p;
  c->stage_pitch[slot] = pitch;
  c->stage_probs_off[slot] = 0;
  c->stage_ploidy_off[slot] = -1;
  return PG_OK;
}

int pg_stage_bgen(pg_ctx* c, int slot, const void* blob, int64_t blob_bytes, const int64_t* block_off,
                  const int64_t* block_size, int64_t count, int64_t* diag) {
  PG_REQUIRE(diag != nullptr, PG_ERR_INVALID, "pg_stage_bgen: null diag");
  PG_CHECK_STATUS(pg_stage_bgen_begin(c, slot, blob, blob_bytes, block_off, block_size, count));
  return pg_stage_bgen_end(c, slot, diag);
}

int pg_scan_staged(pg_ctx* c, int slot, pg_batch_info* info) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(slot == 0 || slot == 1, PG_ERR_INVALID, "pg_scan_staged: slot must be 0 or 1");
  PG_REQUIRE(c->stage_kind[slot] >= 0, PG_ERR_STATE, "pg_scan_staged: slot %d holds no staged batch", slot);
  PG_CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->stage_ev[slot], 0));
  const int kind = c->stage_kind[slot];
  c->stage_kind[slot] = -1;
  const int rc = scan_common(c, kind, c->stage_data[slot], c->stage_m[slot], c->stage_pitch[slot], info,
                             c->stage_probs_off[slot], c->stage_ploidy_off[slot]);
  PG_CUDA_CHECK(cudaEventRecord(c->slot_free_ev[slot], c->stream));
  return rc;
}

int pg_scan_device(pg_ctx* c, int kind, const void* d_data, int64_t n_markers, int64_t row_bytes, int64_t row_pitch,
                   pg_batch_info* info) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_scan_device: no panel uploaded");
  const int64_t expect = expected_row_bytes(kind, c->n_src);
  PG_REQUIRE(expect > 0 && row_bytes == expect, PG_ERR_FORMAT, "row has %lld bytes, expected %lld",
             (long long)row_bytes, (long long)expect);
  PG_REQUIRE(row_pitch % 16 == 0 && row_pitch >= row_bytes, PG_ERR_INVALID, "row_pitch must be a multiple of 16");
  PG_REQUIRE(reinterpret_cast<uintptr_t>(d_data) % 16 == 0, PG_ERR_INVALID, "device block must be 16-byte aligned");
  return scan_common(c, kind, static_cast<const uint8_t*>(d_data), n_markers, row_pitch, info);
}

int pg_time_marker_stats(pg_ctx* c, int kind, const void* d_data, int64_t n_markers, int64_t row_pitch, int reps,
                         float* ms) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_panel, PG_ERR_STATE, "pg_time_marker_stats: no panel uploaded");
  PG_REQUIRE(ms != nullptr && reps >= 1 && n_markers >= 1, PG_ERR_INVALID, "pg_time_marker_stats: bad arguments");
  PG_REQUIRE(row_pitch % 16 == 0 && reinterpret_cast<uintptr_t>(d_data) % 16 == 0, PG_ERR_INVALID,
             "pg_time_marker_stats: rows must be 16-byte aligned");
  GenoBlock b;
  b.kind = kind;
  b.data = static_cast<const uint8_t*>(d_data);
  b.pitch = row_pitch;
  b.n_markers = n_markers;
  b.n_src = c->n_src;
  b.n_kept = c->n_kept;
  b.keep_bits = c->keep_bits.p;
  b.all_kept = c->n_kept == c->n_src ? 1 : 0;
  const int64_t m_cap = round_up(n_markers, 256);
  for (auto* buf : {&c->n_miss, &c->s_u, &c->ss_u}) PG_CHECK_STATUS(buf->ensure(m_cap));
  for (auto* buf : {&c->sum_d, &c->af, &c->var, &c->mu_d, &c->invd_d}) PG_CHECK_STATUS(buf->ensure(m_cap));
  PG_CHECK_STATUS(c->mu_f.ensure(m_cap));
  PG_CHECK_STATUS(c->invd_f.ensure(m_cap));
  PG_CHECK_STATUS(c->skip.ensure(m_cap));
  PG_CHECK_STATUS(c->flags.ensure(2));
  MarkerStats st;
  st.n_miss = c->n_miss.p;
  st.s_u = c->s_u.p;
  st.ss_u = c->ss_u.p;
  st.sum_d = c->sum_d.p;
  st.af = c->af.p;
  st.var = c->var.p;
  st.skip = c->skip.p;
  st.mu_d = c->mu_d.p;
  st.mu_f = c->mu_f.p;
  st.invd_d = c->invd_d.p;
  st.invd_f = c->invd_f.p;
  st.flags = c->flags.p;
  PG_CHECK_STATUS(geno_stats(b, st, m_cap, c->stream));  // warm-up
  PG_CUDA_CHECK(cudaEventRecord(c->ev[0], c->stream));
  for (int i = 0; i < reps; ++i) PG_CHECK_STATUS(geno_stats(b, st, m_cap, c->stream));
  PG_CUDA_CHECK(cudaEventRecord(c->ev[1], c->stream));
  PG_CUDA_CHECK(cudaEventSynchronize(c->ev[1]));
  PG_CUDA_CHECK(cudaEventElapsedTime(ms, c->ev[0], c->ev[1]));
  *ms /= static_cast<float>(reps);
  return PG_OK;
}

int pg_fetch_marker_stats(pg_ctx* c, double* af, int64_t* missing_count, double* variance, int8_t* skip) {
  PG_CHECK_STATUS(ctx_check(c));
  const int64_t m = c->last_m;
  PG_REQUIRE(m > 0, PG_ERR_STATE, "no scanned batch");
  if (af) PG_CUDA_CHECK(cudaMemcpyAsync(af, c->af.p, 8 * m, cudaMemcpyDeviceToHost, c->stream));
  if (missing_count)
    PG_CUDA_CHECK(cudaMemcpyAsync(missing_count, c->n_miss.p, 8 * m, cudaMemcpyDeviceToHost, c->stream));
  if (variance) PG_CUDA_CHECK(cudaMemcpyAsync(variance, c->var.p, 8 * m, cudaMemcpyDeviceToHost, c->stream));
  if (skip) PG_CUDA_CHECK(cudaMemcpyAsync(skip, c->skip.p, m, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_fetch_candidates(pg_ctx* c, int64_t* rows, int64_t* cols, double* r, double* t, double* p) {
  PG_CHECK_STATUS(ctx_check(c));
  const int64_t n = c->last_ncand;
  if (n == 0) return PG_OK;
  if (rows) PG_CUDA_CHECK(cudaMemcpyAsync(rows, c->cand_rows.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  if (cols) PG_CUDA_CHECK(cudaMemcpyAsync(cols, c->cand_cols.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  if (r) PG_CUDA_CHECK(cudaMemcpyAsync(r, c->cand_r_sorted.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  if (t) PG_CUDA_CHECK(cudaMemcpyAsync(t, c->cand_t.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  if (p) PG_CUDA_CHECK(cudaMemcpyAsync(p, c->cand_p.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

namespace {
// FULL rows of the last batch: new_row[m] = output row of non-skipped marker m (-1 skipped)
int full_row_map(pg_ctx* c, const char* who, int elem_bytes, unsigned long long* n_ok) {
  PG_REQUIRE(c->mode == PG_MODE_FULL, PG_ERR_STATE, "%s: ctx not in FULL mode", who);
  PG_REQUIRE(elem_bytes == 4 || elem_bytes == 8, PG_ERR_INVALID, "elem_bytes must be 4 or 8");
  const int64_t m = c->last_m;
  PG_REQUIRE(m > 0, PG_ERR_STATE, "no scanned batch");
  cudaStream_t s = c->stream;
  PG_CHECK_STATUS(c->new_row.ensure(m));
  PG_CUDA_CHECK(cudaMemsetAsync(c->counters.p + 3, 0, sizeof(unsigned long long), s));
  row_map_kernel<<<1, 1024, 0, s>>>(c->skip.p, m, c->new_row.p, c->counters.p + 3);
  PG_CUDA_CHECK(cudaGetLastError());
  PG_CUDA_CHECK(cudaMemcpyAsync(n_ok, c->counters.p + 3, 8, cudaMemcpyDeviceToHost, s));
  PG_CUDA_CHECK(cudaStreamSynchronize(s));
  return PG_OK;
}
}  // namespace

int pg_fetch_full(pg_ctx* c, void* out, int elem_bytes, int64_t* n_rows) {
  PG_CHECK_STATUS(ctx_check(c));
  unsigned long long n_ok = 0;
  PG_CHECK_STATUS(full_row_map(c, "pg_fetch_full", elem_bytes, &n_ok));
  const int64_t m = c->last_m;
  cudaStream_t s = c->stream;
  if (n_rows) *n_rows = static_cast<int64_t>(n_ok);
  if (out == nullptr || n_ok == 0) return PG_OK;
  const size_t bytes = static_cast<size_t>(n_ok) * c->n_pheno * elem_bytes;
  PG_CHECK_STATUS(c->full_out.ensure(bytes));
  PG_CHECK_STATUS(full_rows_to_t(c->full_r.p, m, c->p_pad, c->n_pheno, c->new_row.p, c->df, elem_bytes,
                                 c->full_out.p, c->counters.p, s));
  PG_CUDA_CHECK(cudaMemcpyAsync(out, c->full_out.p, bytes, cudaMemcpyDeviceToHost, s));
  PG_CUDA_CHECK(cudaStreamSynchronize(s));
  return PG_OK;
}

int pg_fetch_full_beta(pg_ctx* c, void* out, int elem_bytes, int64_t* n_rows) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->beta_on, PG_ERR_STATE, "pg_fetch_full_beta: effect sizes not enabled (pg_ctx_set_beta_scale)");
  unsigned long long n_ok = 0;
  PG_CHECK_STATUS(full_row_map(c, "pg_fetch_full_beta", elem_bytes, &n_ok));
  if (n_rows) *n_rows = static_cast<int64_t>(n_ok);
  if (out == nullptr || n_ok == 0) return PG_OK;
  cudaStream_t s = c->stream;
  const size_t bytes = static_cast<size_t>(n_ok) * c->n_pheno * elem_bytes;
  PG_CHECK_STATUS(c->full_out.ensure(bytes));
  PG_CHECK_STATUS(full_rows_to_beta(c->full_r.p, c->last_m, c->p_pad, c->n_pheno, c->new_row.p, c->df, elem_bytes,
                                    c->full_out.p, c->var.p, c->pheno_sd.p, s));
  PG_CUDA_CHECK(cudaMemcpyAsync(out, c->full_out.p, bytes, cudaMemcpyDeviceToHost, s));
  PG_CUDA_CHECK(cudaStreamSynchronize(s));
  return PG_OK;
}

int pg_fetch_candidate_beta(pg_ctx* c, double* beta, double* se) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->beta_on, PG_ERR_STATE,
             "pg_fetch_candidate_beta: effect sizes not enabled (pg_ctx_set_beta_scale)");
  const int64_t n = c->last_ncand;
  if (n == 0) return PG_OK;
  if (beta) PG_CUDA_CHECK(cudaMemcpyAsync(beta, c->cand_beta.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  if (se) PG_CUDA_CHECK(cudaMemcpyAsync(se, c->cand_se.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_fetch_max_abs_r(pg_ctx* c, double* out) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_scan, PG_ERR_STATE, "no scan");
  PG_REQUIRE(c->track_max_abs_r, PG_ERR_STATE, "pg_fetch_max_abs_r: tracking not enabled (pg_ctx_track_max_abs_r)");
  static_assert(sizeof(double) == sizeof(unsigned long long), "fp64 bits");
  PG_CUDA_CHECK(cudaMemcpyAsync(out, c->max_abs_r.p, sizeof(double) * c->n_pheno, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_ctx_track_max_abs_r(pg_ctx* c, int enable) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(c->have_scan, PG_ERR_STATE, "pg_ctx_track_max_abs_r: call after pg_ctx_set_scan");
  c->track_max_abs_r = enable != 0;
  PG_CUDA_CHECK(cudaMemsetAsync(c->max_abs_r.p, 0, sizeof(unsigned long long) * c->p_pad, c->stream));
  return PG_OK;
}

// ---- element-wise statistics (host arrays) ----
int pg_t_from_r(pg_ctx* c, const double* r, int64_t n, double df, double* t) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(df >= 1.0, PG_ERR_INVALID, "t_from_r requires df >= 1");
  if (n <= 0) return PG_OK;
  PG_CHECK_STATUS(c->scratch_a.ensure(n));
  PG_CHECK_STATUS(c->scratch_b.ensure(n));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->scratch_a.p, r, 8 * n, cudaMemcpyHostToDevice, c->stream));
  PG_CHECK_STATUS(elementwise_t_from_r(c->scratch_a.p, n, df, c->scratch_b.p, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(t, c->scratch_b.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_p_from_t(pg_ctx* c, const double* t, int64_t n, double df, double* p, int64_t* underflow) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(df >= 1.0, PG_ERR_INVALID, "p_from_t requires df >= 1");
  if (underflow) *underflow = 0;
  if (n <= 0) return PG_OK;
  PG_CHECK_STATUS(c->scratch_a.ensure(n));
  PG_CHECK_STATUS(c->scratch_b.ensure(n));
  PG_CHECK_STATUS(c->counters.ensure(4));
  PG_CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, 8, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->scratch_a.p, t, 8 * n, cudaMemcpyHostToDevice, c->stream));
  PG_CHECK_STATUS(elementwise_p_from_t(c->scratch_a.p, n, df, c->scratch_b.p, c->counters.p, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(p, c->scratch_b.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  unsigned long long u = 0;
  PG_CUDA_CHECK(cudaMemcpyAsync(&u, c->counters.p, 8, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (underflow) *underflow = static_cast<int64_t>(u);
  return PG_OK;
}

int pg_reg_inc_beta(pg_ctx* c, const double* a, const double* b, const double* x, int64_t n, double* out) {
  PG_CHECK_STATUS(ctx_check(c));
  if (n <= 0) return PG_OK;
  PG_CHECK_STATUS(c->scratch_a.ensure(n));
  PG_CHECK_STATUS(c->scratch_b.ensure(n));
  PG_CHECK_STATUS(c->scratch_c.ensure(n));
  PG_CHECK_STATUS(c->scratch_d.ensure(n));
  PG_CHECK_STATUS(c->flags.ensure(2));
  PG_CUDA_CHECK(cudaMemsetAsync(c->flags.p, 0, 8, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->scratch_a.p, a, 8 * n, cudaMemcpyHostToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->scratch_b.p, b, 8 * n, cudaMemcpyHostToDevice, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(c->scratch_c.p, x, 8 * n, cudaMemcpyHostToDevice, c->stream));
  PG_CHECK_STATUS(
      elementwise_reg_inc_beta(c->scratch_a.p, c->scratch_b.p, c->scratch_c.p, n, c->scratch_d.p, c->flags.p, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(out, c->scratch_d.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  int err = 0;
  PG_CUDA_CHECK(cudaMemcpyAsync(&err, c->flags.p, 4, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  PG_REQUIRE(err == 0, PG_ERR_STATE, "incomplete beta continued fraction did not converge; this is a bug");
  return PG_OK;
}

static int scalar_stat_call(pg_ctx* c, int which, double a, double b, double x, double* out) {
  PG_CHECK_STATUS(c->scratch_a.ensure(1));
  PG_CHECK_STATUS(c->flags.ensure(2));
  PG_CUDA_CHECK(cudaMemsetAsync(c->flags.p, 0, 8, c->stream));
  PG_CHECK_STATUS(scalar_stat(which, a, b, x, c->scratch_a.p, c->flags.p, c->stream));
  int err = 0;
  PG_CUDA_CHECK(cudaMemcpyAsync(out, c->scratch_a.p, 8, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(&err, c->flags.p, 4, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  PG_REQUIRE(err == 0, PG_ERR_STATE, "incomplete beta continued fraction did not converge; this is a bug");
  return PG_OK;
}

int pg_p_from_t_scalar(pg_ctx* c, double t, double df, double* p) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(df >= 1.0, PG_ERR_INVALID, "p_from_t requires df >= 1");
  return scalar_stat_call(c, 1, t, df, 0.0, p);
}

int pg_reg_inc_beta_scalar(pg_ctx* c, double a, double b, double x, double* out) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(a > 0.0 && b > 0.0, PG_ERR_INVALID, "reg_inc_beta requires a > 0 and b > 0");
  PG_REQUIRE(x >= 0.0 && x <= 1.0, PG_ERR_INVALID, "reg_inc_beta requires x in [0, 1]");
  return scalar_stat_call(c, 0, a, b, x, out);
}

int pg_t_threshold_for_p(pg_ctx* c, double p_threshold, double df, double* t_crit) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(p_threshold > 0.0 && p_threshold <= 1.0, PG_ERR_INVALID, "p_threshold must be in (0, 1]");
  PG_REQUIRE(df >= 1.0, PG_ERR_INVALID, "p_from_t requires df >= 1");
  PG_CHECK_STATUS(c->scratch_a.ensure(1));
  PG_CHECK_STATUS(t_threshold(p_threshold, df, c->scratch_a.p, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(t_crit, c->scratch_a.p, 8, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

// ---- genotype decode for the reader API ----
int pg_decode_bed(pg_ctx* c, const uint8_t* packed, int64_t n_markers, int64_t row_bytes, int64_t n_samples,
                  int elem_bytes, void* dosages, int64_t* missing_count) {
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(row_bytes == (n_samples + 3) / 4, PG_ERR_FORMAT,
             "packed row has %lld bytes, expected %lld for %lld samples", (long long)row_bytes,
             (long long)((n_samples + 3) / 4), (long long)n_samples);
  PG_REQUIRE(elem_bytes == 4 || elem_bytes == 8, PG_ERR_INVALID, "elem_bytes must be 4 or 8");
  if (n_markers <= 0) return PG_OK;
  const int64_t pitch = round_up(row_bytes, 16);
  PG_CHECK_STATUS(c->packed.ensure(static_cast<size_t>(pitch) * n_markers));
  PG_CHECK_STATUS(c->full_out.ensure(static_cast<size_t>(n_markers) * n_samples * elem_bytes));
  PG_CHECK_STATUS(c->new_row.ensure(n_markers));
  PG_CHECK_STATUS(upload_rows(packed, n_markers, row_bytes, pitch, c->raw_rows, c->packed.p, c->stream));
  GenoBlock b;
  b.kind = PG_GENO_BED;
  b.data = c->packed.p;
  b.pitch = pitch;
  b.n_markers = n_markers;
  b.n_src = n_samples;
  PG_CHECK_STATUS(geno_dosages(b, elem_bytes, c->full_out.p, c->new_row.p, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(dosages, c->full_out.p, static_cast<size_t>(n_markers) * n_samples * elem_bytes,
                                cudaMemcpyDeviceToHost, c->stream));
  if (missing_count)
    PG_CUDA_CHECK(cudaMemcpyAsync(missing_count, c->new_row.p, 8 * n_markers, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

int pg_decode_bgen(pg_ctx* c, const void* probs_and_ploidy, const uint8_t* unused, int64_t n_markers,
                   int64_t n_samples, int bits, double* dosages, int64_t* missing_count) {
  (void)unused;
  PG_CHECK_STATUS(ctx_check(c));
  PG_REQUIRE(bits == 8 || bits == 16, PG_ERR_INVALID, "bits must be 8 or 16");
  if (n_markers <= 0) return PG_OK;
  const int kind = bits == 8 ? PG_GENO_BGEN8 : PG_GENO_BGEN16;
  const int64_t row_bytes = expected_row_bytes(kind, n_samples);
  const int64_t pitch = round_up(row_bytes, 16);
  PG_CHECK_STATUS(c->packed.ensure(static_cast<size_t>(pitch) * n_markers));
  PG_CHECK_STATUS(c->full_out.ensure(static_cast<size_t>(n_markers) * n_samples * 8));
  PG_CHECK_STATUS(c->new_row.ensure(n_markers));
  PG_CHECK_STATUS(upload_rows(probs_and_ploidy, n_markers, row_bytes, pitch, c->raw_rows, c->packed.p, c->stream));
  GenoBlock b;
  b.kind = kind;
  b.data = c->packed.p;
  b.pitch = pitch;
  b.n_markers = n_markers;
  b.n_src = n_samples;
  PG_CHECK_STATUS(geno_dosages(b, 8, c->full_out.p, c->new_row.p, c->stream));
  PG_CUDA_CHECK(cudaMemcpyAsync(dosages, c->full_out.p, static_cast<size_t>(n_markers) * n_samples * 8,
                                cudaMemcpyDeviceToHost, c->stream));
  if (missing_count)
    PG_CUDA_CHECK(cudaMemcpyAsync(missing_count, c->new_row.p, 8 * n_markers, cudaMemcpyDeviceToHost, c->stream));
  PG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return PG_OK;
}

}  // extern "C"
