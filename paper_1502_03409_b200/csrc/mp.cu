// mp.cu — model parallelism over receptive fields inside the library.
//
// "The training algorithm is model parallel ... distributing the model across the GPUs";
// "Communication within the algorithm occurs when a layer's input (or output) field spans multiple GPUs"
// (PAPER.md:117). The global field grid is cut into tiles_r x tiles_c contiguous rectangles, one per rank in
// row-major order; a rank owns the untied weights of its fields (no weight or gradient
// collective exists) and a pixel rectangle (its fields' window origins; the last tile row / column extends to
// the image edge). Its layer runs on the rectangle its fields read (`need`, owned pixels plus a halo of
// rf - s rows / columns below and to the right). One step:
//
//   C1  input halo: every rank packs the owned pixels its neighbours need (from its internal HWCN image, bf16 on
//       the tensor-core path) and exchanges them with grouped NCCL send / recv on a comm stream; meanwhile the
//       step kernel runs the INTERIOR fields (windows inside the owned pixels) on all but two SM pairs; the
//       BOUNDARY fields run once the halo is unpacked;
//   C2  input-gradient return: the dX of halo pixels (fp32) goes back to their owners, who add it (overlap-add);
//   C3  loss: all-reduce (sum) of the two fp64 loss terms.
//
// Pack / unpack / add are the kernels below (HWCN regions are runs of C*mp contiguous elements per pixel).
// NCCL is loaded at run time (dlopen "libnccl.so.2": the same library torch.distributed uses in-process).
// Test mode (world_size > 1, nccl_id == NULL): no NCCL; the caller moves the exchange buffers between the
// ranks' handles between the three phases of a step (lcae_mp_buffer / lcae_mp_phase), which verifies pack,
// interior / boundary split and overlap-add on one GPU against the untiled layer.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace lcae {

// ------------------------------------------------------------------------------------------------ plan (host)
static void factor(int world, int *tr, int *tc) {   // tiles_r x tiles_c, as square as possible, tiles_r >= tiles_c
  int br = world, bc = 1;
  for (int c = 1; c <= world; ++c)
    if (world % c == 0) {
      const int r = world / c;
      if (r >= c && (r - c) < (br - bc)) { br = r; bc = c; }
    }
  *tr = br;
  *tc = bc;
}

static void split(int n, int parts, int p, int *a, int *b) {   // balanced: the first n % parts get one more
  const int base = n / parts, extra = n % parts;
  *a = p * base + std::min(p, extra);
  *b = *a + base + (p < extra ? 1 : 0);
}

lcae_status mp_tile(const lcae_config *c, const Geo &gg, int rank, MpTile *t) {
  int tr_n = c->tiles_r, tc_n = c->tiles_c;
  if (tr_n <= 0 && tc_n <= 0) factor(c->world_size, &tr_n, &tc_n);
  if (tr_n <= 0 || tc_n <= 0 || tr_n * tc_n != c->world_size) {
    set_error("model parallel: tiles_r * tiles_c must equal world_size");
    return LCAE_ERR_CONFIG;
  }
  if (rank < 0 || rank >= c->world_size) { set_error("model parallel: rank out of range"); return LCAE_ERR_CONFIG; }
  if (tr_n > gg.gr || tc_n > gg.gc) {   // a tile without fields is a configuration error
    set_error("model parallel: more tiles than field rows / columns (a tile would own no field)");
    return LCAE_ERR_CONFIG;
  }
  const int tr = rank / tc_n, tc = rank % tc_n;
  t->tr_n = tr_n;
  t->tc_n = tc_n;
  split(gg.gr, tr_n, tr, &t->R0, &t->R1);
  split(gg.gc, tc_n, tc, &t->C0, &t->C1);
  const int s = gg.s;
  t->need[0] = t->R0 * s;
  t->need[1] = (t->R1 - 1) * s + gg.rf_h;
  t->need[2] = t->C0 * s;
  t->need[3] = (t->C1 - 1) * s + gg.rf_w;
  t->own[0] = t->R0 * s;
  t->own[1] = tr == tr_n - 1 ? gg.H : t->R1 * s;
  t->own[2] = t->C0 * s;
  t->own[3] = tc == tc_n - 1 ? gg.W : t->C1 * s;
  return LCAE_OK;
}

static bool intersect(const int *a, const int *b, int *o) {
  o[0] = std::max(a[0], b[0]);
  o[1] = std::min(a[1], b[1]);
  o[2] = std::max(a[2], b[2]);
  o[3] = std::min(a[3], b[3]);
  return o[0] < o[1] && o[2] < o[3];
}

// ------------------------------------------------------------------------------------------------ kernels
namespace {

// owned NHWC f32 [m][oh][ow][C] -> rows [0, oh) x cols [0, ow) of the HWCN image [Hn][Wn][C][mp] (32 x 32 tiles
// through shared memory; one image row per blockIdx.z); non-finite inputs set flag[0] (include/lcae.h "Errors")
template <typename T>
__global__ void stage_own(const float *__restrict__ x, T *__restrict__ xt, int m, int mp, int oh, int rowlen,
                          int64_t out_row, int *flag) {
  __shared__ float tile[32][33];
  const int y = blockIdx.z, p0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const int64_t in_sample = (int64_t)oh * rowlen;
  bool bad = false;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, p = p0 + threadIdx.x;
    const float v = (i < m && p < rowlen) ? x[(int64_t)i * in_sample + (int64_t)y * rowlen + p] : 0.f;
    bad |= !isfinite(v);
    tile[r][threadIdx.x] = v;
  }
  if (bad) flag[0] = 1;
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int p = p0 + r, i = i0 + threadIdx.x;
    if (i < m && p < rowlen) {
      const float v = tile[threadIdx.x][r];
      T *dst = xt + ((int64_t)y * out_row + p) * mp + i;
      if constexpr (sizeof(T) == 2) *dst = __float2bfloat16_rn(v);
      else *dst = v;
    }
  }
}

// HWCN f32 image rows [0, oh) x cols [0, ow) -> owned NHWC f32 [m][oh][ow][C]
__global__ void unstage_own(const float *__restrict__ xt, float *__restrict__ x, int m, int mp, int oh, int rowlen,
                            int64_t in_row) {
  __shared__ float tile[32][33];
  const int y = blockIdx.z, p0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int p = p0 + r, i = i0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < m && p < rowlen) ? xt[((int64_t)y * in_row + p) * mp + i] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, p = p0 + threadIdx.x;
    if (i < m && p < rowlen) x[(int64_t)i * oh * rowlen + (int64_t)y * rowlen + p] = tile[threadIdx.x][r];
  }
}

// A region of `rows` image rows of `words` 32-bit words each (cols * C * mp elements): pack = strided image ->
// contiguous buffer, unpack = the reverse; add = the image region += the buffer (fp32). Grid-stride, 16-byte
// accesses when both sides are 16-byte aligned.
__global__ void region_copy(uint32_t *__restrict__ img, uint32_t *__restrict__ buf, int rows, int64_t words,
                            int64_t row_pitch_words, int to_buf) {
  const int64_t tot = (int64_t)rows * words;
  const bool v4 = (words & 3) == 0 && (row_pitch_words & 3) == 0 && (((uintptr_t)img | (uintptr_t)buf) & 15) == 0;
  if (v4) {
    const int64_t w4 = words >> 2, t4 = tot >> 2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < t4; t += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = t / w4, q = t - r * w4;
      uint4 *pi = reinterpret_cast<uint4 *>(img + r * row_pitch_words) + q;
      uint4 *pb = reinterpret_cast<uint4 *>(buf) + t;
      if (to_buf) *pb = *pi;
      else *pi = *pb;
    }
    return;
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / words, q = t - r * words;
    if (to_buf) buf[t] = img[r * row_pitch_words + q];
    else img[r * row_pitch_words + q] = buf[t];
  }
}

__global__ void region_add_f32(float *__restrict__ img, const float *__restrict__ buf, int rows, int64_t elems,
                               int64_t row_pitch) {
  const int64_t tot = (int64_t)rows * elems;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / elems, q = t - r * elems;
    img[r * row_pitch + q] += buf[t];
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  void *h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};

static NcclApi *nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.h = h;
#define LCAE_SYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, n))
      LCAE_SYM(getUniqueId, "ncclGetUniqueId");
      LCAE_SYM(commInitRank, "ncclCommInitRank");
      LCAE_SYM(commDestroy, "ncclCommDestroy");
      LCAE_SYM(send, "ncclSend");
      LCAE_SYM(recv, "ncclRecv");
      LCAE_SYM(groupStart, "ncclGroupStart");
      LCAE_SYM(groupEnd, "ncclGroupEnd");
      LCAE_SYM(allReduce, "ncclAllReduce");
      LCAE_SYM(errStr, "ncclGetErrorString");
#undef LCAE_SYM
    }
  }
  return api.h && api.send && api.recv && api.commInitRank && api.allReduce ? &api : nullptr;
}

#define LCAE_NCCL(call)                                                                          \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess) {                                                                     \
      set_error(std::string("NCCL: ") + #call + ": " + (nccl()->errStr ? nccl()->errStr(r_) : "")); \
      return LCAE_ERR_NCCL;                                                                      \
    }                                                                                            \
  } while (0)

// ------------------------------------------------------------------------------------------------ state
struct MpRegion {
  int peer;
  int ly0, ly1, lx0, lx1;   // in this rank's local (need-region) pixel coordinates
  size_t off, elems;        // in the exchange buffer (elements of the buffer's type)
};

struct MpState {
  MpTile t;
  int world = 1, rank = 0;
  bool use_nccl = false;
  ncclComm_t comm = nullptr;
  std::vector<MpRegion> in_send, in_recv;   // input halo (C1): owned pixels out / needed pixels in
  size_t in_send_n = 0, in_recv_n = 0, px_elems = 0;   // px_elems = C * mp per pixel
  void *in_send_buf = nullptr, *in_recv_buf = nullptr;   // element type of the internal image (bf16 / f32)
  float *dx_send_buf = nullptr, *dx_recv_buf = nullptr;   // C2: same regions, fp32, reversed direction
  int *flist = nullptr;
  int n_int = 0, n_bnd = 0;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_staged = nullptr, ev_halo = nullptr;
  int phase = 0;   // test mode: next expected phase
};

static size_t elem_size(lcae_layer *L) { return L->cfg.precision == LCAE_FP32 ? 4 : 2; }
static void *image(lcae_layer *L) { return L->cfg.precision == LCAE_FP32 ? (void *)L->xt32 : (void *)L->xt16; }

lcae_status mp_init(lcae_layer *L, const Geo &gg) {
  MpState *M = new MpState();
  L->mpst = M;
  const lcae_config &c = L->cfg;
  M->world = c.world_size;
  M->rank = c.rank;
  LCAE_CK(cudaGetLastError());
  lcae_status st = mp_tile(&c, gg, c.rank, &M->t);
  if (st) return st;
  const Geo &g = L->geo;   // local (need region)
  M->px_elems = (size_t)g.C * L->mp;
  // regions: for every other rank b, C1 sends intersect(b.need, my own) and receives intersect(my need, b.own);
  // C2 (dX) runs the same regions in the opposite direction
  for (int b = 0; b < M->world; ++b) {
    if (b == M->rank) continue;
    MpTile tb;
    if ((st = mp_tile(&c, gg, b, &tb))) return st;
    int r[4];
    if (intersect(tb.need, M->t.own, r)) {
      MpRegion q{b, r[0] - M->t.need[0], r[1] - M->t.need[0], r[2] - M->t.need[2], r[3] - M->t.need[2], M->in_send_n, 0};
      q.elems = (size_t)(r[1] - r[0]) * (r[3] - r[2]) * M->px_elems;
      M->in_send_n += q.elems;
      M->in_send.push_back(q);
    }
    if (intersect(M->t.need, tb.own, r)) {
      MpRegion q{b, r[0] - M->t.need[0], r[1] - M->t.need[0], r[2] - M->t.need[2], r[3] - M->t.need[2], M->in_recv_n, 0};
      q.elems = (size_t)(r[1] - r[0]) * (r[3] - r[2]) * M->px_elems;
      M->in_recv_n += q.elems;
      M->in_recv.push_back(q);
    }
  }
  const size_t es = elem_size(L);
  if (M->in_send_n) {
    LCAE_CK(dmalloc(L, &M->in_send_buf, M->in_send_n * es));
    LCAE_CK(dmalloc(L, &M->dx_recv_buf, M->in_send_n * 4));
  }
  if (M->in_recv_n) {
    LCAE_CK(dmalloc(L, &M->in_recv_buf, M->in_recv_n * es));
    LCAE_CK(dmalloc(L, &M->dx_send_buf, M->in_recv_n * 4));
  }
  // interior fields (window inside the owned pixels: computable before the halo arrives), then boundary fields
  const int oh = M->t.own[1] - M->t.own[0], ow = M->t.own[3] - M->t.own[2];
  std::vector<int> fl;
  for (int pass = 0; pass < 2; ++pass)
    for (int f = 0; f < g.F; ++f) {
      const int r = f / g.gc, cc = f % g.gc;
      const bool inside = r * g.s + g.rf_h <= oh && cc * g.s + g.rf_w <= ow;
      if (inside == (pass == 0)) fl.push_back(f);
      if (pass == 0 && inside) ++M->n_int;
    }
  M->n_bnd = g.F - M->n_int;
  LCAE_CK(dmalloc(L, &M->flist, fl.size() * sizeof(int)));
  LCAE_CK(cudaMemcpy(M->flist, fl.data(), fl.size() * sizeof(int), cudaMemcpyHostToDevice));
  LCAE_CK(cudaStreamCreateWithFlags(&M->cs, cudaStreamNonBlocking));
  LCAE_CK(cudaEventCreateWithFlags(&M->ev_staged, cudaEventDisableTiming));
  LCAE_CK(cudaEventCreateWithFlags(&M->ev_halo, cudaEventDisableTiming));
  M->use_nccl = c.nccl_id != nullptr;
  if (M->use_nccl) {
    NcclApi *api = nccl();
    if (!api) { set_error("model parallel: libnccl.so.2 could not be loaded"); return LCAE_ERR_NCCL; }
    ncclUniqueId id;
    memcpy(&id, c.nccl_id, sizeof id);
    LCAE_NCCL(api->commInitRank(&M->comm, M->world, id, M->rank));
  }
  return LCAE_OK;
}

void mp_free(lcae_layer *L) {
  MpState *M = L->mpst;
  if (!M) return;
  if (M->comm && nccl() && nccl()->commDestroy) nccl()->commDestroy(M->comm);
  for (void *p : {M->in_send_buf, M->in_recv_buf, (void *)M->dx_send_buf, (void *)M->dx_recv_buf, (void *)M->flist})
    if (p) cudaFree(p);
  if (M->cs) cudaStreamDestroy(M->cs);
  if (M->ev_staged) cudaEventDestroy(M->ev_staged);
  if (M->ev_halo) cudaEventDestroy(M->ev_halo);
  delete M;
  L->mpst = nullptr;
}

// pack (to_buf) / unpack a list of regions of the internal image (elements of size es) on `st`
static lcae_status move_regions(lcae_layer *L, const std::vector<MpRegion> &rs, void *img, void *buf, size_t es,
                                bool to_buf, cudaStream_t st) {
  const Geo &g = L->geo;
  const MpState *M = L->mpst;
  for (const MpRegion &q : rs) {
    const size_t pxw = M->px_elems * es / 4;   // 32-bit words per pixel
    uint32_t *ip = reinterpret_cast<uint32_t *>(img) + ((size_t)q.ly0 * g.W + q.lx0) * pxw;
    uint32_t *bp = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(buf) + q.off * es);
    region_copy<<<L->sm_count * 2, 256, 0, st>>>(ip, bp, q.ly1 - q.ly0, (int64_t)(q.lx1 - q.lx0) * pxw,
                                                (int64_t)g.W * pxw, to_buf ? 1 : 0);
    LCAE_CK_LAUNCH(L);
  }
  return LCAE_OK;
}

// one grouped NCCL exchange: send `sends` regions of sbuf, receive `recvs` regions into rbuf (byte granularity)
static lcae_status exchange(lcae_layer *L, const std::vector<MpRegion> &sends, const void *sbuf,
                            const std::vector<MpRegion> &recvs, void *rbuf, size_t es, cudaStream_t st) {
  MpState *M = L->mpst;
  NcclApi *api = nccl();
  LCAE_NCCL(api->groupStart());
  for (const MpRegion &q : sends)
    LCAE_NCCL(api->send(reinterpret_cast<const char *>(sbuf) + q.off * es, q.elems * es, ncclUint8, q.peer, M->comm, st));
  for (const MpRegion &q : recvs)
    LCAE_NCCL(api->recv(reinterpret_cast<char *>(rbuf) + q.off * es, q.elems * es, ncclUint8, q.peer, M->comm, st));
  LCAE_NCCL(api->groupEnd());
  return LCAE_OK;
}

size_t mp_input_elems(lcae_layer *L) {
  const MpTile &t = L->mpst->t;
  return (size_t)L->geo.m * (t.own[1] - t.own[0]) * (t.own[3] - t.own[2]) * L->geo.C;
}

// owned NHWC f32 (device) -> the internal image's owned rows / columns
lcae_status mp_stage(lcae_layer *L, const float *xd) {
  const Geo &g = L->geo;
  const MpTile &t = L->mpst->t;
  const int oh = t.own[1] - t.own[0], rowlen = (t.own[3] - t.own[2]) * g.C;
  dim3 grid((unsigned)cdiv(rowlen, 32), (unsigned)cdiv(g.m, 32), (unsigned)oh);
  if (L->cfg.precision == LCAE_FP32)
    stage_own<float><<<grid, dim3(32, 8), 0, L->st>>>(xd, L->xt32, g.m, L->mp, oh, rowlen, (int64_t)g.W * g.C,
                                                      L->flags_dev);
  else
    stage_own<__nv_bfloat16><<<grid, dim3(32, 8), 0, L->st>>>(xd, L->xt16, g.m, L->mp, oh, rowlen,
                                                              (int64_t)g.W * g.C, L->flags_dev);
  LCAE_CK_LAUNCH(L);
  return LCAE_OK;
}

// Phases of a model-parallel step (NCCL mode runs all three inside lcae_step / lcae_forward):
//  0: (x staged by the caller) pack the halo others need; NCCL: exchange it on the comm stream and unpack as it
//     lands; run the interior fields (bf16) concurrently;
//  1: (test mode: unpack the halo the caller delivered) boundary fields (bf16) / all fields (fp32, general bf16
//     path), finalize,
//     local loss; pack the dX of halo pixels for their owners;
//  2: (NCCL: exchange dX) add the returned dX into the owned pixels; all-reduce the loss (NCCL).
lcae_status mp_phase(lcae_layer *L, int phase, bool update, bool want_pooled) {
  MpState *M = L->mpst;
  const size_t es = elem_size(L);
  const bool bf16 = L->cfg.precision == LCAE_BF16 && !L->gt;   // the fused kernel (interior / boundary launches)
  lcae_status s;
  if (phase == 0) {
    if ((s = move_regions(L, M->in_send, image(L), M->in_send_buf, es, true, L->st))) return s;
    if (M->use_nccl) {
      LCAE_CK(cudaEventRecord(M->ev_staged, L->st));
      LCAE_CK(cudaStreamWaitEvent(M->cs, M->ev_staged, 0));
      if ((s = exchange(L, M->in_send, M->in_send_buf, M->in_recv, M->in_recv_buf, es, M->cs))) return s;
      if ((s = move_regions(L, M->in_recv, image(L), M->in_recv_buf, es, false, M->cs))) return s;
      LCAE_CK(cudaEventRecord(M->ev_halo, M->cs));
    }
    if (update) LCAE_CK(cudaMemsetAsync(L->dxt, 0, (size_t)L->geo.H * L->geo.W * L->geo.C * L->mp * 4, L->st));
    if (bf16 && M->n_int)
      return tc_step(L, update, want_pooled, false, M->flist, M->n_int, false, false, M->use_nccl ? 2 : 0);
    return LCAE_OK;
  }
  if (phase == 1) {
    if (M->use_nccl) LCAE_CK(cudaStreamWaitEvent(L->st, M->ev_halo, 0));
    else if ((s = move_regions(L, M->in_recv, image(L), M->in_recv_buf, es, false, L->st))) return s;
    if (bf16) s = tc_step(L, update, want_pooled, false, M->flist + M->n_int, M->n_bnd, false, true, 0);
    else if (L->gt) s = gt_step(L, update, want_pooled, false);   // general bf16 path: every field after the halo
    else s = f32_step(L, update, want_pooled);
    if (s) return s;
    if ((s = launch_loss_reduce(L, update))) return s;
    if (update && (s = move_regions(L, M->in_recv, L->dxt, M->dx_send_buf, 4, true, L->st))) return s;
    return LCAE_OK;
  }
  // phase 2
  if (update) {
    if (M->use_nccl && (s = exchange(L, M->in_recv, M->dx_send_buf, M->in_send, M->dx_recv_buf, 4, L->st))) return s;
    const Geo &g = L->geo;
    for (const MpRegion &q : M->in_send) {   // dX of my owned pixels computed by the ranks that read them
      float *ip = L->dxt + ((size_t)q.ly0 * g.W + q.lx0) * M->px_elems;
      region_add_f32<<<L->sm_count * 2, 256, 0, L->st>>>(ip, M->dx_recv_buf + q.off, q.ly1 - q.ly0,
                                                         (int64_t)(q.lx1 - q.lx0) * M->px_elems,
                                                         (int64_t)g.W * M->px_elems);
      LCAE_CK_LAUNCH(L);
    }
    const MpTile &t = M->t;
    const int oh = t.own[1] - t.own[0], rowlen = (t.own[3] - t.own[2]) * g.C;
    dim3 grid((unsigned)cdiv(rowlen, 32), (unsigned)cdiv(g.m, 32), (unsigned)oh);
    unstage_own<<<grid, dim3(32, 8), 0, L->st>>>(L->dxt, L->dx_nhwc, g.m, L->mp, oh, rowlen, (int64_t)g.W * g.C);
    LCAE_CK_LAUNCH(L);
  }
  if (M->use_nccl) LCAE_NCCL(nccl()->allReduce(L->loss_dev, L->loss_dev, 2, ncclFloat64, ncclSum, M->comm, L->st));
  return LCAE_OK;
}

bool mp_external(lcae_layer *L) { return L->mpst && !L->mpst->use_nccl; }

lcae_status mp_buffer(lcae_layer *L, int which, int peer, void **ptr, int64_t *bytes) {
  MpState *M = L->mpst;
  const std::vector<MpRegion> &rs = (which == 0 || which == 3) ? M->in_send : M->in_recv;
  const size_t es = which < 2 ? elem_size(L) : 4;
  char *base = reinterpret_cast<char *>(which == 0 ? M->in_send_buf : which == 1 ? M->in_recv_buf
                                        : which == 2 ? (void *)M->dx_send_buf : (void *)M->dx_recv_buf);
  for (const MpRegion &q : rs)
    if (q.peer == peer) {
      if (ptr) *ptr = base + q.off * es;
      if (bytes) *bytes = (int64_t)(q.elems * es);
      return LCAE_OK;
    }
  if (ptr) *ptr = nullptr;
  if (bytes) *bytes = 0;
  return LCAE_OK;
}

void mp_counts(lcae_layer *L, int *n_int, int *n_bnd) {
  *n_int = L->mpst->n_int;
  *n_bnd = L->mpst->n_bnd;
}

const MpTile &mp_tile_of(lcae_layer *L) { return L->mpst->t; }

}  // namespace lcae

extern "C" lcae_status lcae_nccl_unique_id(void *out128) {
  if (!out128) { lcae::set_error("NULL argument"); return LCAE_ERR_ARG; }
  lcae::NcclApi *api = lcae::nccl();
  if (!api || !api->getUniqueId) { lcae::set_error("libnccl.so.2 could not be loaded"); return LCAE_ERR_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = api->getUniqueId(&id);
  if (r != ncclSuccess) {
    lcae::set_error(std::string("ncclGetUniqueId: ") + (api->errStr ? api->errStr(r) : ""));
    return LCAE_ERR_NCCL;
  }
  memcpy(out128, &id, sizeof id);
  return LCAE_OK;
}
