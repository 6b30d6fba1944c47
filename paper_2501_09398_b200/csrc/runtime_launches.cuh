// runtime_launches.cuh — per-iteration kernel launch lists: vector, hotspot variants, FDTD (k_fdtd_lf modes, lean fallback, slabs, ranks).
// Part of runtime.cu (one translation unit; included in order, not compiled alone).
#pragma once

namespace {

int64_t numel(const int64_t *s, int n) {
  int64_t r = 1;
  for (int i = 0; i < n; ++i) r *= s[i];
  return r;
}

// ---- per-iteration launch lists ----------------------------------------------------------------
int hotspot_rows_per_chunk(const ib_ctx *c, int rows) {
  int64_t rpc = env_int("IB_HOTSPOT_RPC", 0);
  if (rpc <= 0) {
    const int64_t want_threads = 148LL * 2048 * 2;
    int64_t chunks = (want_threads + c->plane() - 1) / c->plane();
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, rows));
    rpc = (rows + chunks - 1) / chunks;
    rpc = std::min<int64_t>(rpc, 64);
  }
  // grid.y = ceil(rows / rpc) must stay <= 65535 (tall, narrow grids: e.g. 100000 x 4)
  rpc = std::max<int64_t>(rpc, (rows + 65534) / 65535);
  return (int)std::max<int64_t>(1, std::min<int64_t>(rpc, rows));
}

// Kernel variant for a hotspot grid. IB_HOTSPOT_KERNEL=scalar|vec|tma forces one (if legal).
//   vec    one 16-byte group per thread, every load independent: best for L2-resident grids
//   tma    cp.async.bulk plane-march pipeline: best once the state no longer fits in L2
//   scalar marching fallback for shapes the vector paths cannot take (M or L not a multiple of V)
enum class HotKernel { Scalar, Vec, Tma };

template <typename T>
int tma_groups(const ib_ctx *c) {  // G such that TM = G*V*256 holds whole y-rows; 0 = not possible
  constexpr int V = 16 / sizeof(T);
  const bool d3 = c->solver == IB_SOLVER_HOTSPOT3D;
  const int64_t L = d3 ? c->dims[2] : 1;
  const int64_t force = env_int("IB_TMA_GROUPS", 0);  // tuning: 1, 2 or 4 groups per thread
  for (int G : {2, 1, 4}) {
    if (force > 0 && G != force) continue;
    const int64_t TM = (int64_t)G * V * 256;
    if (!d3 || (TM % L == 0 && L <= 1024)) return G;
  }
  return 0;
}

template <typename T>
HotKernel hotspot_variant(const ib_ctx *c, int g, int rows) {
  constexpr int V = 16 / sizeof(T);
  const bool d3 = c->solver == IB_SOLVER_HOTSPOT3D;
  const int64_t M = c->plane();
  const int64_t L = d3 ? c->dims[2] : 1;
  const bool vec_ok = (M % V == 0) && (!d3 || L % V == 0) && rows <= 65535 &&
                      (int64_t)(rows + 2) * M < (1LL << 31);  // 32-bit offsets
  const bool tma_ok = vec_ok && tma_groups<T>(c) > 0 && rows >= 2;
  const char *force = env_str("IB_HOTSPOT_KERNEL");
  if (force) {
    if (!std::strcmp(force, "tma") && tma_ok) return HotKernel::Tma;
    if (!std::strcmp(force, "vec") && vec_ok) return HotKernel::Vec;
    if (!std::strcmp(force, "scalar")) return HotKernel::Scalar;
  }
  // the bytes that share this slab's L2: every slab on the same device, halo planes included
  // (one rank of a multi-process run holds only its own slab)
  int64_t planes = 0;
  const bool multi = c->slabs.size() > 1 || c->dist();
  for (const Slab &s : c->slabs)
    if (s.device == c->slabs[g].device) planes += s.rows() + (multi ? 2 : 0);
  if (planes == 0) planes = rows;
  const int64_t state_bytes = 3 * M * planes * (int64_t)sizeof(T);
  // the state (T twice + P) against the 126 MB L2: measured crossover (tools/hotspot_vec_vs_tma.py,
  // us/iter vec / tma): 3-D 1024^2x8 (100.7 MB) 16.3 / 19.0, 1280x1024x8 (126 MB) 22.6 / 22.5,
  // 1536x1024x8 27.1 / 25.7; 2-D 2048^2 (50 MB) 8.3 / 8.9, 3072^2 (113 MB) 19.3 / 18.0.
  if (tma_ok && state_bytes >= (104LL << 20)) return HotKernel::Tma;
  if (vec_ok) return HotKernel::Vec;
  return HotKernel::Scalar;
}

template <typename T, bool D3>
const void *tma_fn(int G) {
  switch (G) {
    case 1: return (const void *)ib::k_hotspot_tma<T, D3, 1>;
    case 4: return (const void *)ib::k_hotspot_tma<T, D3, 4>;
    default: return (const void *)ib::k_hotspot_tma<T, D3, 2>;
  }
}

template <typename T, bool D3, int SH, bool FS>
const void *vec_fn_r(int R) {
  return R >= 4 ? (const void *)ib::k_hotspot_vec<T, D3, 4, SH, FS>
         : R == 2 ? (const void *)ib::k_hotspot_vec<T, D3, 2, SH, FS>
                  : (const void *)ib::k_hotspot_vec<T, D3, 1, SH, FS>;
}
template <typename T, bool FS>
const void *vec_fn_f(bool d3, int R, int sh) {
  if (d3) return sh == 2 ? vec_fn_r<T, true, 2, FS>(R) : sh == 1 ? vec_fn_r<T, true, 1, FS>(R) : vec_fn_r<T, true, 0, FS>(R);
  return sh ? vec_fn_r<T, false, 1, FS>(R) : vec_fn_r<T, false, 0, FS>(R);
}
// fs: the cross-process peer exchange's system-scope fence after halo stores (kernels.cuh)
template <typename T>
const void *vec_fn(bool d3, int R, int sh, bool fs) {
  return fs ? vec_fn_f<T, true>(d3, R, sh) : vec_fn_f<T, false>(d3, R, sh);
}

template <typename T>
void hotspot_launches(ib_ctx *c, int parity, std::vector<Launch> &out) {
  constexpr int V = 16 / sizeof(T);
  const bool d3 = c->solver == IB_SOLVER_HOTSPOT3D;
  const int C = (int)c->dims[1];
  const int L = d3 ? (int)c->dims[2] : 1;
  const int64_t plane = c->plane();
  const T k = (T)c->scalars[0];
  const T loss = (T)(2.0 * (d3 ? 3 : 2));
  const int P = (int)c->slabs.size();
  const bool multi = P > 1 || c->dist();  // slab buffers carry halo planes
  for (int g = 0; g < P; ++g) {
    Slab &s = c->slabs[g];
    const int rows = s.rows();
    const int64_t off = multi ? plane : 0;  // first owned plane
    const T *src = (const T *)s.buf[parity] + off;
    T *dst = (T *)s.buf[parity ^ 1] + off;
    T *up = nullptr, *dn = nullptr;
    if (P > 1 && g > 0 && !c->halo_copy) {  // my first owned row -> upper neighbour's bottom halo
      Slab &n = c->slabs[g - 1];
      up = (T *)n.buf[parity ^ 1] + (int64_t)(n.rows() + 1) * plane;
    }
    if (P > 1 && g + 1 < P && !c->halo_copy) {  // my last owned row -> lower neighbour's top halo
      Slab &n = c->slabs[g + 1];
      dn = (T *)n.buf[parity ^ 1];
    }
    if (c->dist() && c->peer) {  // the neighbour ranks' halo planes, through IPC mappings
      if (s.has_top) up = (T *)c->peer_buf_up[parity ^ 1] + (int64_t)(c->peer_rows_up + 1) * plane;
      if (s.has_bot) dn = (T *)c->peer_buf_dn[parity ^ 1];
    }
    const int top = (int)s.has_top, bot = (int)s.has_bot;
    const int fsys = (int)(c->dist() && c->peer);  // system-scope fence after halo stores (kernels.cuh)
    dim3 block(256);
    switch (hotspot_variant<T>(c, g, rows)) {
      case HotKernel::Vec: {
        // rows per thread (R+2 row loads per R outputs): with the neighbour loads (no shuffles)
        // R = 1 — the most threads, the shortest per-thread chain — unless the grid would exceed
        // four waves (measured: Hotspot3D 512x512x8 R=1 4.41, R=2 4.57, R=4 4.67 us/iter;
        // Hotspot2D 1024^2 R=1 2.56, R=2 3.12); with shuffles R = 2 (below). IB_HOTSPOT_VEC_ROWS
        // overrides.
        int64_t R = env_int("IB_HOTSPOT_VEC_ROWS", 0);
        const int64_t threads_per_row = plane / V;
        // CTA shape: bx threads along a plane row (up to 256), by row-blocks, bx*by = IB_HOTSPOT_BLOCK.
        // 256 measured best in-graph (Hotspot3D 512^2x8: 4.45 / 4.79 / 6.20 us at 256 / 512 / 1024;
        // Hotspot2D 2.60 / 2.65 / 2.68) although an EMPTY kernel's launch floor falls with fewer,
        // bigger CTAs (tools/microbench_floor.cu): real CTAs retire at their slowest warp.
        // With shuffles and R = 2 (below), 2-D measured best at 512 threads (256 x 2 row-blocks:
        // 2.33 vs 2.43 us/iter at 256), 3-D at 256 (4.21; 512: 4.61).
        // 3-D grids of >= 2^19 groups with whole-warp rows (Hotspot3D 512^2x8): 4 rows per thread
        // in 128 x 8-thread CTAs measured 2% faster than 2 rows in 256 x 1 (4.10 vs 4.20 us/iter,
        // interleaved repeats, tools/hotspot3d_repeat.py; tools/cta_shape_tune.py swept the rest).
        // Only while those 1024-thread CTAs (one per SM at <= 64 registers) fit in one wave:
        // 768x512x8 (192 CTAs) ran 30% slower than the 256 x 1 shape.
        const bool wide3d = d3 && threads_per_row * rows >= (1LL << 19) && threads_per_row % 32 == 0 &&
                            32 % (L / V) == 0 &&
                            ((threads_per_row + 127) / 128) * ((rows + 31) / 32) <= c->num_sms;
        // binary64 3-D (two cells per 16-byte group, so twice the threads of binary32 for a grid):
        // 4 rows per thread in 128-thread CTAs measured best — Hotspot3D 512^2x8 6.57 us/iter
        // against 7.31 for the 256-thread / R = 2 binary32 default, 6.70-6.72 for R = 4 / 256 and
        // R = 2 / 128 (tools/hotspot_tune.py, DTYPE=f64, graph with PDL edges)
        const bool d3_f64 = d3 && sizeof(T) == 8 && !wide3d;
        // binary64 2-D (Hotspot2D 1024^2, the headline config): 64 x 8-thread CTAs, whose 8 rows
        // share their x-neighbour rows in L1, and the in-row neighbours loaded instead of shuffled
        // (a double needs two SHFL.32) — 3.56 us/iter against 3.92 for the binary32 shape (256 x 2,
        // shuffles, R = 2 -> 1); every other 2-D / 3-D shape of either precision measured within
        // 1% of its default (tools/hotspot_vec_shapes.py, profiles/r02_hotspot_vec_shapes.md)
        const bool d2_f64 = !d3 && sizeof(T) == 8;
        int64_t bs = env_int("IB_HOTSPOT_BLOCK", d3 ? (wide3d ? 1024 : (d3_f64 ? 128 : 256)) : 512);
        bs = std::max<int64_t>(32, std::min<int64_t>(1024, bs / 32 * 32));
        const int64_t bx_max =
            std::max<int64_t>(32, env_int("IB_HOTSPOT_BX", wide3d ? 128 : (d2_f64 ? 64 : 256)) / 32 * 32);  // CTA width cap
        const int64_t bx = std::min<int64_t>(std::min<int64_t>(bx_max, bs), (threads_per_row + 31) / 32 * 32);
        const int64_t by = std::max<int64_t>(1, bs / bx);
        const int64_t xblocks = (threads_per_row + bx - 1) / bx;
        if (R <= 0) {
          const int64_t slots = 1536LL * c->num_sms;  // resident threads at <= 40 registers
          R = 1;
          while (R < 4 && xblocks * bx * ((rows + R - 1) / R) > 4 * slots) R *= 2;
        }
        R = R >= 4 ? 4 : (R >= 2 ? 2 : 1);
        // warp shuffles for the in-row (2-D) / z (3-D) neighbours when every warp covers 32 groups
        // of one row and whole y-rows: 1 = those, 2 = also the y rows. IB_HOTSPOT_SHUFFLE overrides.
        const int64_t gl = d3 ? L / V : 1;
        // Measured in-graph with PDL (us/iter, two runs): Hotspot3D 512^2x8 R=1 4.47, R=1+sh1 4.36,
        // R=2+sh1 4.22-4.25, sh2 (y rows by 8 shuffles) 4.60-4.77; Hotspot2D 1024^2 R=1 2.61,
        // R=1+sh1 2.49, R=2+sh1 2.45. So z / row shuffles, and 2 rows per thread with them.
        int64_t sh = env_int("IB_HOTSPOT_SHUFFLE", d2_f64 ? 0 : 1);
        if (!(threads_per_row % 32 == 0 && bx % 32 == 0 && 32 % gl == 0)) sh = 0;
        if (sh && env_int("IB_HOTSPOT_VEC_ROWS", 0) <= 0 && rows >= 2 && R < 2) R = 2;
        if ((wide3d || d3_f64) && sh && env_int("IB_HOTSPOT_VEC_ROWS", 0) <= 0 && rows >= 4) R = 4;
        // 2-D grids past one wave of the 256 x 2 / R = 2 shape (two 512-thread CTAs per SM at 49
        // registers): one row per thread (~30 registers, four CTAs per SM) measured faster —
        // 2048^2 7.89 vs 8.67 us/iter, 1536^2 5.92 vs 6.75 (tools/hotspot2d_shapes.py)
        if (!d3 && sh && env_int("IB_HOTSPOT_VEC_ROWS", 0) <= 0 && R == 2 &&
            xblocks * ((rows + 2 * by - 1) / (2 * by)) > 2LL * c->num_sms)
          R = 1;
        const void *fn = vec_fn<T>(d3, (int)R, (int)std::min<int64_t>(sh, 2), fsys != 0);
        dim3 grid((unsigned)xblocks, (unsigned)((rows + R * by - 1) / (R * by)));
        out.push_back(make_launch(fn, grid, dim3((unsigned)bx, (unsigned)by), g, src, dst, (const T *)s.power,
                                  rows, C, L, k, loss,
                                  top, bot, up, dn));
        break;
      }
      case HotKernel::Tma: {
        const int G = tma_groups<T>(c);
        const int TM = G * V * 256;
        const int H = d3 ? L : V;
        const int ns = (int)std::max<int64_t>(3, std::min<int64_t>(8, env_int("IB_TMA_STAGES", 4)));
        const size_t smem = (size_t)ns * (TM + 2 * H + TM) * sizeof(T) + (size_t)ns * 8;
        const void *fn = d3 ? tma_fn<T, true>(G) : tma_fn<T, false>(G);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t tiles = (plane + TM - 1) / TM;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
        const int64_t slots = (int64_t)std::max(1, per_sm) * c->num_sms;
        int64_t rpc = env_int("IB_HOTSPOT_RPC", 0);
        if (rpc <= 0) {
          rpc = std::max<int64_t>(16, std::min<int64_t>(128, (int64_t)rows * tiles / (12 * slots)));
          // Few waves: a partial last wave idles most SMs for a whole CTA's march (Hotspot2D 4096^2:
          // 512 CTAs on 444 slots), so round the grid to whole waves (>= 8 rows per CTA).
          const int64_t ctas = tiles * ((rows + rpc - 1) / rpc);
          if (ctas < 3 * slots) {
            const int64_t waves = std::max<int64_t>(1, (ctas + slots / 2) / slots);
            const int64_t chunks = std::max<int64_t>(1, waves * slots / tiles);
            rpc = std::max<int64_t>(8, (rows + chunks - 1) / chunks);
          }
        }
        rpc = std::min<int64_t>(rpc, rows);
        dim3 grid((unsigned)tiles, (unsigned)((rows + rpc - 1) / rpc));
        Launch Lz = make_launch(fn, grid, block, g, src, dst, (const T *)s.power, rows, C, L, (int)rpc, ns,
                                k, loss, top, bot, up, dn, fsys);
        Lz.smem = smem;
        out.push_back(Lz);
        break;
      }
      default: {
        const void *fn = d3 ? (const void *)ib::k_hotspot<T, true> : (const void *)ib::k_hotspot<T, false>;
        const int rpc = hotspot_rows_per_chunk(c, rows);
        dim3 grid((unsigned)((plane + 255) / 256), (unsigned)((rows + rpc - 1) / rpc));
        out.push_back(make_launch(fn, grid, block, g, src, dst, (const T *)s.power, rows, C, L, rpc, k,
                                  loss, top, bot, up, dn, fsys));
      }
    }
  }
}

// Fused leapfrog (k_fdtd_lf): TJ y-rows per tile, NS-stage bulk-copy ring. The largest TJ (and
// then NS) whose ring lets two CTAs share an SM; the grid is one wave of resident CTAs and the
// (tile, plane) units are split evenly over it. IB_FDTD_TJ / IB_FDTD_STAGES override.
struct LfConfig {
  int tj = 0, ns = 0;
  size_t smem = 0;
};
inline size_t lf_smem(int tj, int ns, int64_t P, int es) {
  return (size_t)ns * (size_t)(3 * (tj + 2) + 3 * (tj + 1)) * (size_t)P * es + (size_t)ns * 8;
}
inline int lf_threads(const ib_ctx *c, int tj) {  // one thread per (row, 16-byte group)
  const int64_t groups = c->lat_pitch / (16 / c->esize);
  return (int)(((tj + 1) * groups + 31) / 32 * 32);
}
// short_run: a binary32 H or E launch over <= 40 planes (an axis-0 slab of 256^3 split 8 ways):
// 3-row tiles with a 4-stage ring, two CTAs per SM, measured best there — 35-plane slab 27.8 vs
// 32.1 us per H+E iteration (the default shape spends a larger share of a short launch filling
// its deeper ring), equal at 67 planes and slower beyond (tools/fdtd_slab_tune.py,
// profiles/r02_slab_scaling.md)
inline LfConfig lf_config(const ib_ctx *c, bool short_run = false) {
  // The kernel is bound by how much each SM keeps in flight, and the ring depth in planes counts
  // more than its bytes. Measured at 256^3 (us/iter) binary32: TJ=4/NS=6 one CTA per SM 130.7,
  // TJ=4/NS=5 137.3, TJ=3/NS=4 two per SM 138.5, TJ=3/NS=3 196, TJ=4/NS=3 171; binary64 (twice
  // the threads per row): TJ=2/NS=5 fused 300.6 / two half-steps 383.4, TJ=3/NS=4 364 / 480,
  // TJ=4/NS=3 433 / 486. So: the first shape (largest tiles, one CTA per SM first) whose ring
  // holds >= 5 stages, else >= 4, else any. IB_FDTD_TJ / IB_FDTD_STAGES force a shape.
  const int64_t P = c->lat_pitch;
  const int es = c->esize;
  const size_t cap = 227 * 1024, half = 113 * 1024;
  const int64_t ftj = env_int("IB_FDTD_TJ", 0), fns = env_int("IB_FDTD_STAGES", 0);
  if (short_run && ftj <= 0 && fns <= 0 && es == 4 && lf_threads(c, 3) <= ib::kLfNarrowThreads &&
      lf_smem(3, 4, P, es) <= half)
    return LfConfig{3, 4, lf_smem(3, 4, P, es)};
  const struct { int tj; bool two; } order[] = {{4, false}, {3, true}, {4, true}, {2, true},
                                                 {3, false}, {2, false}, {1, true}, {1, false}};
  for (int min_ns : {5, 4, 3}) {
    for (auto o : order) {
      if (ftj > 0 && o.tj != ftj) continue;
      if (lf_threads(c, o.tj) > ib::lf_max_threads(es)) continue;
      LfConfig cfg;
      for (int ns = 3; ns <= (fns > 0 ? 12 : 6); ++ns) {
        if (fns > 0 && ns != fns) continue;
        const size_t sm = lf_smem(o.tj, ns, P, es);
        if (sm <= (o.two ? half : cap)) cfg = {o.tj, ns, sm};
      }
      if (cfg.tj && (cfg.ns >= min_ns || fns > 0)) return cfg;
    }
  }
  return LfConfig{};
}

template <typename T, bool U, int M, bool W>
const void *lf_fn_w(int tj) {
  switch (tj) {
    case 1: return (const void *)ib::k_fdtd_lf<T, U, 1, M, W>;
    case 2: return (const void *)ib::k_fdtd_lf<T, U, 2, M, W>;
    case 3: return (const void *)ib::k_fdtd_lf<T, U, 3, M, W>;
    default: return (const void *)ib::k_fdtd_lf<T, U, 4, M, W>;
  }
}
template <typename T, bool U, int M>
const void *lf_fn_m(int tj, bool wide) { return wide ? lf_fn_w<T, U, M, true>(tj) : lf_fn_w<T, U, M, false>(tj); }
template <typename T, bool U>
const void *lf_fn_u(int tj, int mode, bool wide) {
  switch (mode) {
    case ib::kLfH: return lf_fn_m<T, U, ib::kLfH>(tj, wide);
    case ib::kLfE: return lf_fn_m<T, U, ib::kLfE>(tj, wide);
    case ib::kLfFusedSlab: return lf_fn_m<T, U, ib::kLfFusedSlab>(tj, wide);
    default: return lf_fn_m<T, U, ib::kLfFused>(tj, wide);
  }
}
template <typename T>
const void *lf_fn(bool unit, int tj, int mode, bool wide) {
  return unit ? lf_fn_u<T, true>(tj, mode, wide) : lf_fn_u<T, false>(tj, mode, wide);
}

// One k_fdtd_lf launch of `mode` from lattice buffer `from` to `to` (equal for the in-place
// half-steps).
template <typename T>
Launch lf_launch(ib_ctx *c, int mode, void *from, void *to, int x0, int npl, int64_t fs, void *halo_h = nullptr,
                 int64_t fs_h = 0, void *halo_e = nullptr, int64_t fs_e = 0, int slab = 0) {
  const int nx = (int)c->dims[0], ny = (int)c->dims[1], nz = (int)c->dims[2];
  const T d = (T)c->scalars[0], ch = (T)c->scalars[1], ce = (T)c->scalars[2];
  const bool unit = c->scalars[0] == 1.0;
  const LfConfig cfg = lf_config(c, (mode == ib::kLfH || mode == ib::kLfE) && npl <= 40);
  const int threads = lf_threads(c, cfg.tj);
  const void *fn = lf_fn<T>(unit, cfg.tj, mode, threads > ib::kLfNarrowThreads);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, cfg.smem);
  // Lockstep (tile, x-chunk) grid: as many x-chunks as the resident slots hold whole columns of
  // TJ-row tiles (256^3, TJ=4, 148 slots: 65 tiles x 2 chunks). Filling the spare slots with
  // shorter tiles (74 tiles of 3-4 rows x 2) measured slower (137 vs 131 us): more halo rows.
  // IB_FDTD_TILES (uneven rows, h <= TJ), IB_FDTD_CHUNKS, IB_FDTD_CTAS (even split) override.
  const int64_t slots = (int64_t)std::max(1, per_sm) * c->num_sms;
  const int64_t min_tiles = (ny + 1 + cfg.tj - 1) / cfg.tj;
  int64_t tiles = min_tiles;
  if (env_int("IB_FDTD_TILES", 0) >= min_tiles) tiles = std::min<int64_t>(ny + 1, env_int("IB_FDTD_TILES", 0));
  int64_t chunks = env_int("IB_FDTD_CHUNKS", 0);
  if (chunks <= 0) chunks = std::max<int64_t>(1, slots / tiles);
  chunks = std::min<int64_t>(chunks, npl);  // every chunk non-empty
  int64_t ctas = env_int("IB_FDTD_CTAS", 0);
  if (ctas <= 0 && env_int("IB_FDTD_CHUNKS", 0) <= 0 && tiles > slots) ctas = slots;  // > one wave of
  // tiles (long rows force short tiles, e.g. 384^3): one wave, the unit list split evenly
  if (ctas <= 0) {
    ctas = tiles * chunks;  // one CTA per (tile, chunk): the kernel maps blockIdx.x to both
  } else {
    chunks = 0;  // even split of the tile-major unit list over `ctas` CTAs
    ctas = std::max<int64_t>(1, std::min(ctas, tiles * npl));
  }
  Launch L = make_launch(fn, dim3((unsigned)ctas), dim3((unsigned)threads), slab, (const T *)from, (T *)to, nx,
                         ny, nz, (int)c->lat_pitch, fs, x0, npl, (int)tiles, (int)chunks, cfg.ns, ch, ce, d,
                         (T *)halo_h, fs_h, (T *)halo_e, fs_e, (int)(c->dist() && c->peer));
  L.smem = cfg.smem;
  L.step = mode == ib::kLfE ? 1 : 0;
  return L;
}

// FDTD, the reference's two half-steps (H then E, in place on the lattice): k_fdtd_lf in its H
// and E modes, or the lean one-thread-per-point kernels when the z rows are too long for the
// staged kernel's CTA (or IB_FDTD_KERNEL=lean).
template <typename T>
void fdtd_launches(ib_ctx *c, std::vector<Launch> &out) {
  // The staged kernel marches planes serially per CTA; while the lattice sits in L2 the fully
  // parallel lean kernels finish sooner. Round 2, vectorised lean vs staged (us/iter, binary32 /
  // binary64, tools/lean_vs_staged.py): 96^3 11.7 / 17.8 and 17.4 / 25.0, 128^3 25.5 / 27.3 and
  // 54.5 / 48.3 (107 MB lattice), 144^3 33.1 / 44.6, 160^3 56.6 / 62.8, 192^3 94.8 / 89.9, 256^3
  // 221 / 202 and 385 / 382 — so lean while the lattice is below 104 MB (the hotspot kernels'
  // L2 crossover too). IB_FDTD_KERNEL=lean|staged.
  // Long z rows leave the staged kernel only 1-row tiles or a 3-stage ring (binary64 384^3: TJ=1 /
  // NS=4 2,508 us/iter, TJ=2 / NS=3 2,042, against 1,408 for the lean kernels: 0.90 of the copy
  // peak; profiles/r02_size_sweep.md, tools/fdtd_tune.py) — the lean kernels take those shapes too.
  const char *force = env_str("IB_FDTD_KERNEL");
  const int64_t lattice_bytes = 6 * c->lat_fs * c->esize;
  const LfConfig cfg = lf_config(c);
  const bool shallow = cfg.tj <= 1 || cfg.ns <= 3;
  const bool lean = (force && !std::strcmp(force, "lean")) || cfg.tj == 0 ||
                    (!force && shallow && env_int("IB_FDTD_TJ", 0) <= 0 && env_int("IB_FDTD_STAGES", 0) <= 0) ||
                    (!force && c->slabs.size() == 1 && !c->dist() && lattice_bytes < (104LL << 20));
  const int nx = (int)c->dims[0];
  const int P = (int)c->slabs.size();
  if (c->dist()) {  // one rank's slab; the neighbours' halo planes through IPC mappings
    const int64_t plane = (int64_t)(c->dims[1] + 1) * c->lattice_pitch();
    Slab &s = c->slabs[0];
    T *base = (T *)s.buf[0] + (int64_t)(1 - s.row_lo) * plane;
    void *hh = nullptr, *he = nullptr;
    int64_t fh = 0, fe = 0;
    if (c->peer && s.has_bot) {
      hh = c->peer_buf_dn[0];  // the down rank's top halo plane (its local 0)
      fh = (int64_t)(c->peer_rows_dn + 2) * plane;
    }
    if (c->peer && s.has_top) {
      he = (T *)c->peer_buf_up[0] + (int64_t)(c->peer_rows_up + 1) * plane;  // the up rank's bottom halo
      fe = (int64_t)(c->peer_rows_up + 2) * plane;
    }
    out.push_back(lf_launch<T>(c, ib::kLfH, base, base, s.row_lo, s.rows(), s.fs, hh, fh, nullptr, 0, 0));
    out.push_back(lf_launch<T>(c, ib::kLfE, base, base, s.row_lo, s.rows(), s.fs, nullptr, 0, he, fe, 0));
    return;
  }
  if (P > 1) {  // axis-0 slabs: every H launch, then every E launch, halo planes pushed in-kernel
    const int64_t plane = (int64_t)(c->dims[1] + 1) * c->lat_pitch;
    for (int step = 0; step < 2; ++step)
      for (int g = 0; g < P; ++g) {
        Slab &s = c->slabs[g];
        T *base = (T *)s.buf[0] + (int64_t)(1 - s.row_lo) * plane;  // global plane index -> buffer
        void *hh = nullptr, *he = nullptr;
        int64_t fh = 0, fe = 0;
        if (step == 0 && g + 1 < P && !c->halo_copy) {  // IB_HALO_COPY: copy nodes instead
          hh = c->slabs[g + 1].buf[0];  // its top halo plane (local 0)
          fh = c->slabs[g + 1].fs;
        }
        if (step == 1 && g > 0 && !c->halo_copy) {
          Slab &n = c->slabs[g - 1];
          he = (T *)n.buf[0] + (int64_t)(n.rows() + 1) * plane;  // its bottom halo plane
          fe = n.fs;
        }
        out.push_back(lf_launch<T>(c, step == 0 ? ib::kLfH : ib::kLfE, base, base, s.row_lo, s.rows(), s.fs,
                                   hh, fh, he, fe, g));
      }
    return;
  }
  if (!lean) {
    out.push_back(lf_launch<T>(c, ib::kLfH, c->lat[0], c->lat[0], 0, nx + 1, c->lat_fs));
    out.push_back(lf_launch<T>(c, ib::kLfE, c->lat[0], c->lat[0], 0, nx + 1, c->lat_fs));
    return;
  }
  const int ny = (int)c->dims[1], nz = (int)c->dims[2];
  const T d = (T)c->scalars[0], ch = (T)c->scalars[1], ce = (T)c->scalars[2];
  const bool unit = c->scalars[0] == 1.0;
  dim3 b2(32, 8);
  // one 16-byte group per thread (k_fdtd_h4 / e4) — measured faster than one cell per thread
  // (k_fdtd_h2 / e2) wherever HBM matters (us/iter, scalar / vector: binary32 256^3 277 / 224,
  // 96x256x720 245 / 209, binary64 256^3 432 / 390, 384^3 1379 / 1264), equal on small binary32
  // grids and 9% slower on small binary64 ones (64^3 8.7 / 9.5), which keep the scalar pair
  // (tools/lean_ab.py). IB_FDTD_LEANV=0|1 forces one.
  const int64_t leanv = env_int("IB_FDTD_LEANV", -1);
  const bool vec = leanv >= 0 ? leanv != 0 : !(c->esize == 8 && lattice_bytes < (32LL << 20));
  constexpr int V = 16 / sizeof(T);
  dim3 grid((unsigned)(vec ? (c->lat_pitch / V + 31) / 32 : (nz + 1 + 31) / 32), (unsigned)((ny + 1 + 7) / 8),
            (unsigned)(nx + 1));
  const void *fh = vec ? (unit ? (const void *)ib::k_fdtd_h4<T, true> : (const void *)ib::k_fdtd_h4<T, false>)
                       : (unit ? (const void *)ib::k_fdtd_h2<T, true> : (const void *)ib::k_fdtd_h2<T, false>);
  const void *fe = vec ? (unit ? (const void *)ib::k_fdtd_e4<T, true> : (const void *)ib::k_fdtd_e4<T, false>)
                       : (unit ? (const void *)ib::k_fdtd_e2<T, true> : (const void *)ib::k_fdtd_e2<T, false>);
  T *f = (T *)c->lat[0];
  out.push_back(make_launch(fh, grid, b2, 0, f, nx, ny, nz, (int)c->lat_pitch, c->lat_fs, ch, d));
  out.push_back(make_launch(fe, grid, b2, 0, f, nx, ny, nz, (int)c->lat_pitch, c->lat_fs, ce, d));
  out.back().step = 1;
}

// FDTD fused: one k_fdtd_lf launch per iteration, parity -> parity ^ 1.
template <typename T>
void fdtd_fused_launches(ib_ctx *c, int parity, std::vector<Launch> &out) {
  const int P = (int)c->slabs.size();
  if (P == 1 && !c->dist()) {
    out.push_back(lf_launch<T>(c, ib::kLfFused, c->lat[parity], c->lat[parity ^ 1], 0, (int)c->dims[0] + 1,
                               c->lat_fs));
    return;
  }
  // axis-0 slabs of the lattice, ping-pong per slab: slab g reads buf[parity] (its planes and the
  // halo plane each side) and writes buf[parity ^ 1]; its kernel stores its last plane's new E and
  // H into slab g+1's lower halo (that slab's seed plane) and its first plane's new E into slab
  // g-1's upper halo (the E_old(i+1) of that slab's last plane), both in buf[parity ^ 1].
  const int64_t plane = (int64_t)(c->dims[1] + 1) * c->lattice_pitch();
  if (c->dist()) {  // one rank's slab; the neighbour ranks' buffers through IPC mappings
    Slab &s = c->slabs[0];
    const int64_t off = (int64_t)(1 - s.row_lo) * plane;
    void *hh = nullptr, *he = nullptr;
    int64_t fh = 0, fe = 0;
    if (c->peer && s.has_bot) {
      hh = c->peer_buf_dn[parity ^ 1];  // the down rank's lower halo plane (its local 0)
      fh = (int64_t)(c->peer_rows_dn + 2) * plane;
    }
    if (c->peer && s.has_top) {
      he = (T *)c->peer_buf_up[parity ^ 1] + (int64_t)(c->peer_rows_up + 1) * plane;  // its upper halo
      fe = (int64_t)(c->peer_rows_up + 2) * plane;
    }
    out.push_back(lf_launch<T>(c, ib::kLfFusedSlab, (T *)s.buf[parity] + off, (T *)s.buf[parity ^ 1] + off,
                               s.row_lo, s.rows(), s.fs, hh, fh, he, fe, 0));
    return;
  }
  for (int g = 0; g < P; ++g) {
    Slab &s = c->slabs[g];
    const int64_t off = (int64_t)(1 - s.row_lo) * plane;  // global plane index addresses the buffer
    T *src = (T *)s.buf[parity] + off, *dst = (T *)s.buf[parity ^ 1] + off;
    void *hh = nullptr, *he = nullptr;
    int64_t fh = 0, fe = 0;
    if (g + 1 < P && !c->halo_copy) {  // IB_HALO_COPY: copy nodes instead (runtime_graphs.cuh)
      Slab &n = c->slabs[g + 1];
      hh = n.buf[parity ^ 1];  // its lower halo plane (local 0)
      fh = n.fs;
    }
    if (g > 0 && !c->halo_copy) {
      Slab &n = c->slabs[g - 1];
      he = (T *)n.buf[parity ^ 1] + (int64_t)(n.rows() + 1) * plane;  // its upper halo plane
      fe = n.fs;
    }
    out.push_back(lf_launch<T>(c, ib::kLfFusedSlab, src, dst, s.row_lo, s.rows(), s.fs, hh, fh, he, fe, g));
  }
}

void iteration_launches(ib_ctx *c, int parity, std::vector<Launch> &out) {
  out.clear();
  switch (c->solver) {
    case IB_SOLVER_VECTOR: {
      const int64_t n = c->dims[0];
      const double cc = c->scalars[0];
      // Small vectors (the skeleton, 2^14): one item per thread in 128-thread CTAs (measured best:
      // 1.21 / 1.23 / 1.24 / 1.40 us per iteration at 128 / 256 / 512 / 1024). Beyond one wave of
      // threads CTA dispatch dominates (~1.2 ns per CTA: 8192 CTAs for 2^22 elements), so
      // 1024-thread CTAs, two per SM, grid-stride. IB_VECTOR_BLOCK overrides the block size.
      const int64_t items = c->dtype == IB_F32 ? (n >> 2) + (n & 3) : (n >> 1) + (n & 1);
      const bool big = items > 2048LL * c->num_sms;
      int64_t bs = env_int("IB_VECTOR_BLOCK", big ? 1024 : 128);
      bs = std::max<int64_t>(32, std::min<int64_t>(1024, bs / 32 * 32));
      const int64_t cap_ctas = big ? 2LL * c->num_sms * (2048 / bs) / 2 : 8LL * c->num_sms * (2048 / bs);
      if (c->dtype == IB_F32) {
        const int64_t threads = (n >> 2) + (n & 3), need = (threads + bs - 1) / bs;
        dim3 block((unsigned)bs), grid((unsigned)std::min<int64_t>(cap_ctas, need));
        const void *fn = need > cap_ctas ? (const void *)ib::k_vector_f32<true> : (const void *)ib::k_vector_f32<false>;
        out.push_back(make_launch(fn, grid, block, 0, (float *)c->field[0], n, cc));
      } else {
        const int64_t threads = (n >> 1) + (n & 1), need = (threads + bs - 1) / bs;
        dim3 block((unsigned)bs), grid((unsigned)std::min<int64_t>(cap_ctas, need));
        const void *fn = need > cap_ctas ? (const void *)ib::k_vector_f64<true> : (const void *)ib::k_vector_f64<false>;
        out.push_back(make_launch(fn, grid, block, 0, (double *)c->field[0], n, cc));
      }
      break;
    }
    case IB_SOLVER_HOTSPOT2D:
    case IB_SOLVER_HOTSPOT3D:
      if (c->dtype == IB_F32)
        hotspot_launches<float>(c, parity, out);
      else
        hotspot_launches<double>(c, parity, out);
      break;
    case IB_SOLVER_FDTD:
      if (c->dtype == IB_F32)
        fdtd_launches<float>(c, out);
      else
        fdtd_launches<double>(c, out);
      break;
    case IB_SOLVER_FDTD_FUSED:
      if (c->dtype == IB_F32)
        fdtd_fused_launches<float>(c, parity, out);
      else
        fdtd_fused_launches<double>(c, parity, out);
      break;
  }
}

}  // namespace
