/*
 * ib_oracle.c — CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library, and only as the checker or the timed CPU baseline — never as the product.
 * The product (paper_2501_09398_b200/) never links or calls it and has no CPU fallback.
 *
 * It restates, op for op, the numpy arithmetic of /root/reference/pkg/src/iterbatch/workloads.py
 * in the same STRUCTURE as the reference (explicit edge padding, out-of-place H step, copy + interior
 * update + wall zeroing for E) rather than the fused in-place form the CUDA kernels use, so that
 * agreement between the two is evidence and not a tautology. Each numpy binary op is one C binary op
 * on the same type; the recipe (oracle/Makefile) builds with -ffp-contract=off -fno-fast-math, and
 * x86-64 SSE arithmetic is correctly rounded in binary32 and binary64, which is what numpy does.
 *
 * Pinned: tests/test_oracle.py checks the binary64 build against the golden checksums and fixtures in
 * tests/golden/ that tests/golden/make_golden.py produced by running the reference itself.
 *
 * Functions (T = f64 | f32):
 *   or_vector_T   workloads.py:97-105   v = v * c   (f32: v = (float)((double)v * c))
 *   or_hotspot_T  workloads.py:167-207  np.pad(edge) + per-axis pair grouping, loss = 2*dims
 *   or_fdtd_T     workloads.py:325-413  fdtd_h_step then fdtd_e_step, `steps` times
 *   or_fnv1a64    workloads.py:508-517  64-bit FNV-1a
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

uint64_t or_fnv1a64(const void *data, size_t n, uint64_t h) {
  const unsigned char *p = (const unsigned char *)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* workloads.py:520-525: hash of the "<f8" bytes; binary32 values are widened exactly first. */
uint64_t or_fnv1a64_f32_as_f64(const float *v, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) {
    double d = (double)v[i];
    h = or_fnv1a64(&d, 8, h);
  }
  return h;
}

/* ---- skeleton: vector_scale_step, workloads.py:97-105 ------------------------------------- */
void or_vector_f64(double *v, int64_t n, double c, int64_t steps) {
  for (int64_t s = 0; s < steps; ++s) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) v[i] = v[i] * c; /* out[lo:hi] = w.values[lo:hi] * c */
  }
}

void or_vector_f32(float *v, int64_t n, double c, int64_t steps) {
  for (int64_t s = 0; s < steps; ++s) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) v[i] = (float)((double)v[i] * c);
  }
}

/* ---- hotspot_step, workloads.py:167-207 ------------------------------------------------------
 * padded = np.pad(temp, 1, mode="edge")                                         (177)
 * 2-D: out = center + k * ((x_pair + y_pair) - loss * center) + power           (182-185)
 * 3-D: out = center + k * (((x_pair + y_pair) + z_pair) - loss * center) + power (188-204)
 * Python evaluates  a + k*b + p  as  (a + (k*b)) + p.
 * L == 1 with dims == 2 is the 2-D grid (R, C).                                                */
#define OR_HOTSPOT(T, NAME)                                                                        \
  void NAME(T *temp, const T *power, int64_t R, int64_t C, int64_t L, int dims, T k,             \
            int64_t steps) {                                                                     \
    const int three = dims == 3;                                                                 \
    const int64_t PR = R + 2, PC = C + 2, PL = three ? L + 2 : 1;                                \
    T *pad = (T *)malloc(sizeof(T) * (size_t)(PR * PC * PL));                                    \
    const T loss = (T)(2.0 * dims);                                                              \
    for (int64_t s = 0; s < steps; ++s) {                                                        \
      /* edge padding: padded[a,b,c] = temp[clamp(a-1), clamp(b-1), clamp(c-1)] */               \
      _Pragma("omp parallel for schedule(static)") for (int64_t a = 0; a < PR; ++a) {            \
        int64_t ia = a - 1 < 0 ? 0 : (a - 1 >= R ? R - 1 : a - 1);                              \
        for (int64_t b = 0; b < PC; ++b) {                                                       \
          int64_t ib = b - 1 < 0 ? 0 : (b - 1 >= C ? C - 1 : b - 1);                             \
          for (int64_t c = 0; c < PL; ++c) {                                                     \
            int64_t ic = three ? (c - 1 < 0 ? 0 : (c - 1 >= L ? L - 1 : c - 1)) : 0;             \
            pad[(a * PC + b) * PL + c] = temp[(ia * C + ib) * L + ic];                           \
          }                                                                                      \
        }                                                                                        \
      }                                                                                          \
      _Pragma("omp parallel for schedule(static)") for (int64_t i = 0; i < R; ++i) {             \
        for (int64_t j = 0; j < C; ++j) {                                                        \
          for (int64_t l = 0; l < L; ++l) {                                                      \
            const int64_t pl = three ? l + 1 : 0;                                                \
            const T center = pad[((i + 1) * PC + (j + 1)) * PL + pl];                            \
            const T x_pair = pad[((i)*PC + (j + 1)) * PL + pl] + pad[((i + 2) * PC + (j + 1)) * PL + pl]; \
            const T y_pair = pad[((i + 1) * PC + (j)) * PL + pl] + pad[((i + 1) * PC + (j + 2)) * PL + pl]; \
            T acc = x_pair + y_pair;                                                             \
            if (three) {                                                                         \
              const T z_pair = pad[((i + 1) * PC + (j + 1)) * PL + (pl - 1)] +                   \
                               pad[((i + 1) * PC + (j + 1)) * PL + (pl + 1)];                    \
              acc = acc + z_pair;                                                                \
            }                                                                                    \
            const T lc = loss * center;                                                          \
            const T q = acc - lc;                                                                \
            const T kq = k * q;                                                                  \
            const T r = center + kq;                                                             \
            temp[(i * C + j) * L + l] = r + power[(i * C + j) * L + l];                          \
          }                                                                                      \
        }                                                                                        \
      }                                                                                          \
    }                                                                                            \
    free(pad);                                                                                   \
  }

OR_HOTSPOT(double, or_hotspot_f64)
OR_HOTSPOT(float, or_hotspot_f32)

/* ---- FDTD, workloads.py:325-413 ---------------------------------------------------------------
 * Shapes: ex (nx,ny+1,nz+1) ey (nx+1,ny,nz+1) ez (nx+1,ny+1,nz)
 *         hx (nx+1,ny,nz)   hy (nx,ny+1,nz)   hz (nx,ny,nz+1)
 * H step (out of place, as the reference allocates new hx/hy/hz):
 *   hx = w.hx + c_h*((ey[:,:,1:]-ey[:,:,:-1])/d - (ez[:,1:,:]-ez[:,:-1,:])/d)        (335-338)
 *   hy = w.hy + c_h*((ez[1:,:,:]-ez[:-1,:,:])/d - (ex[:,:,1:]-ex[:,:,:-1])/d)        (341-344)
 *   hz = w.hz + c_h*((ex[:,1:,:]-ex[:,:-1,:])/d - (ey[1:,:,:]-ey[:-1,:,:])/d)        (347-350)
 * E step (copy, interior update from the ORIGINAL E, then zero tangential walls):     (367-412)   */
#define IX(a, b, c, B, Cc) (((int64_t)(a) * (B) + (b)) * (Cc) + (c))

#define OR_FDTD(T, NAME)                                                                           \
  void NAME(T *ex, T *ey, T *ez, T *hx, T *hy, T *hz, int64_t nx, int64_t ny, int64_t nz, T d,    \
            T c_h, T c_e, int64_t steps) {                                                       \
    const size_t n_hx = (size_t)((nx + 1) * ny * nz), n_hy = (size_t)(nx * (ny + 1) * nz),       \
                 n_hz = (size_t)(nx * ny * (nz + 1));                                            \
    const size_t n_ex = (size_t)(nx * (ny + 1) * (nz + 1)),                                      \
                 n_ey = (size_t)((nx + 1) * ny * (nz + 1)),                                      \
                 n_ez = (size_t)((nx + 1) * (ny + 1) * nz);                                      \
    T *nhx = (T *)malloc(sizeof(T) * n_hx), *nhy = (T *)malloc(sizeof(T) * n_hy),                \
      *nhz = (T *)malloc(sizeof(T) * n_hz);                                                      \
    T *nex = (T *)malloc(sizeof(T) * n_ex), *ney = (T *)malloc(sizeof(T) * n_ey),                \
      *nez = (T *)malloc(sizeof(T) * n_ez);                                                      \
    for (int64_t s = 0; s < steps; ++s) {                                                        \
      /* ---- fdtd_h_step ---- */                                                                \
      _Pragma("omp parallel for schedule(static)") for (int64_t i = 0; i < nx + 1; ++i)          \
        for (int64_t j = 0; j < ny; ++j)                                                         \
          for (int64_t k = 0; k < nz; ++k) {                                                     \
            T a = (ey[IX(i, j, k + 1, ny, nz + 1)] - ey[IX(i, j, k, ny, nz + 1)]) / d;           \
            T b = (ez[IX(i, j + 1, k, ny + 1, nz)] - ez[IX(i, j, k, ny + 1, nz)]) / d;           \
            nhx[IX(i, j, k, ny, nz)] = hx[IX(i, j, k, ny, nz)] + c_h * (a - b);                  \
          }                                                                                      \
      _Pragma("omp parallel for schedule(static)") for (int64_t i = 0; i < nx; ++i)              \
        for (int64_t j = 0; j < ny + 1; ++j)                                                     \
          for (int64_t k = 0; k < nz; ++k) {                                                     \
            T a = (ez[IX(i + 1, j, k, ny + 1, nz)] - ez[IX(i, j, k, ny + 1, nz)]) / d;           \
            T b = (ex[IX(i, j, k + 1, ny + 1, nz + 1)] - ex[IX(i, j, k, ny + 1, nz + 1)]) / d;   \
            nhy[IX(i, j, k, ny + 1, nz)] = hy[IX(i, j, k, ny + 1, nz)] + c_h * (a - b);          \
          }                                                                                      \
      _Pragma("omp parallel for schedule(static)") for (int64_t i = 0; i < nx; ++i)              \
        for (int64_t j = 0; j < ny; ++j)                                                         \
          for (int64_t k = 0; k < nz + 1; ++k) {                                                 \
            T a = (ex[IX(i, j + 1, k, ny + 1, nz + 1)] - ex[IX(i, j, k, ny + 1, nz + 1)]) / d;   \
            T b = (ey[IX(i + 1, j, k, ny, nz + 1)] - ey[IX(i, j, k, ny, nz + 1)]) / d;           \
            nhz[IX(i, j, k, ny, nz + 1)] = hz[IX(i, j, k, ny, nz + 1)] + c_h * (a - b);          \
          }                                                                                      \
      memcpy(hx, nhx, sizeof(T) * n_hx);                                                         \
      memcpy(hy, nhy, sizeof(T) * n_hy);                                                         \
      memcpy(hz, nhz, sizeof(T) * n_hz);                                                         \
      /* ---- fdtd_e_step: ex = w.ex.copy() ... ---- */                                          \
      memcpy(nex, ex, sizeof(T) * n_ex);                                                         \
      memcpy(ney, ey, sizeof(T) * n_ey);                                                         \
      memcpy(nez, ez, sizeof(T) * n_ez);                                                         \
      /* ex[:, 1:-1, 1:-1] = w.ex + c_e*((hz[:,1:,1:-1]-hz[:,:-1,1:-1])/d - (hy[:,1:-1,1:]-hy[:,1:-1,:-1])/d) */ \
      _Pragma("omp parallel for schedule(static)") for (int64_t i = 0; i < nx; ++i)              \
        for (int64_t j = 1; j < ny; ++j)                                                         \
          for (int64_t k = 1; k < nz; ++k) {                                                     \
            T a = (hz[IX(i, j, k, ny, nz + 1)] - hz[IX(i, j - 1, k, ny, nz + 1)]) / d;           \
            T b = (hy[IX(i, j, k, ny + 1, nz)] - hy[IX(i, j, k - 1, ny + 1, nz)]) / d;           \
            nex[IX(i, j, k, ny + 1, nz + 1)] = ex[IX(i, j, k, ny + 1, nz + 1)] + c_e * (a - b);  \
          }                                                                                      \
      /* ey[1:nx, :, 1:-1] = w.ey + c_e*((hx[..,1:]-hx[..,:-1])/d - (hz[i]-hz[i-1])/d)  (378-385) */ \
      _Pragma("omp parallel for schedule(static)") for (int64_t i = 1; i < nx; ++i)              \
        for (int64_t j = 0; j < ny; ++j)                                                         \
          for (int64_t k = 1; k < nz; ++k) {                                                     \
            T a = (hx[IX(i, j, k, ny, nz)] - hx[IX(i, j, k - 1, ny, nz)]) / d;                   \
            T b = (hz[IX(i, j, k, ny, nz + 1)] - hz[IX(i - 1, j, k, ny, nz + 1)]) / d;           \
            ney[IX(i, j, k, ny, nz + 1)] = ey[IX(i, j, k, ny, nz + 1)] + c_e * (a - b);          \
          }                                                                                      \
      /* ez[1:nx, 1:-1, :] = w.ez + c_e*((hy[i]-hy[i-1])/d - (hx[:,1:,:]-hx[:,:-1,:])/d) (387-394) */ \
      _Pragma("omp parallel for schedule(static)") for (int64_t i = 1; i < nx; ++i)              \
        for (int64_t j = 1; j < ny; ++j)                                                         \
          for (int64_t k = 0; k < nz; ++k) {                                                     \
            T a = (hy[IX(i, j, k, ny + 1, nz)] - hy[IX(i - 1, j, k, ny + 1, nz)]) / d;           \
            T b = (hx[IX(i, j, k, ny, nz)] - hx[IX(i, j - 1, k, ny, nz)]) / d;                   \
            nez[IX(i, j, k, ny + 1, nz)] = ez[IX(i, j, k, ny + 1, nz)] + c_e * (a - b);          \
          }                                                                                      \
      /* conducting walls: tangential E pinned to zero (400-412) */                               \
      for (int64_t i = 0; i < nx; ++i)                                                           \
        for (int64_t j = 0; j < ny + 1; ++j)                                                     \
          for (int64_t k = 0; k < nz + 1; ++k)                                                   \
            if (j == 0 || j == ny || k == 0 || k == nz) nex[IX(i, j, k, ny + 1, nz + 1)] = (T)0.0; \
      for (int64_t i = 0; i < nx + 1; ++i)                                                       \
        for (int64_t j = 0; j < ny; ++j)                                                         \
          for (int64_t k = 0; k < nz + 1; ++k)                                                   \
            if (i == 0 || i == nx || k == 0 || k == nz) ney[IX(i, j, k, ny, nz + 1)] = (T)0.0;   \
      for (int64_t i = 0; i < nx + 1; ++i)                                                       \
        for (int64_t j = 0; j < ny + 1; ++j)                                                     \
          for (int64_t k = 0; k < nz; ++k)                                                       \
            if (i == 0 || i == nx || j == 0 || j == ny) nez[IX(i, j, k, ny + 1, nz)] = (T)0.0;   \
      memcpy(ex, nex, sizeof(T) * n_ex);                                                         \
      memcpy(ey, ney, sizeof(T) * n_ey);                                                         \
      memcpy(ez, nez, sizeof(T) * n_ez);                                                         \
    }                                                                                            \
    free(nhx);                                                                                   \
    free(nhy);                                                                                   \
    free(nhz);                                                                                   \
    free(nex);                                                                                   \
    free(ney);                                                                                   \
    free(nez);                                                                                   \
  }

OR_FDTD(double, or_fdtd_f64)
OR_FDTD(float, or_fdtd_f32)
