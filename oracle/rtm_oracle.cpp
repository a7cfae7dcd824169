// =====================================================================================
//  ORACLE — TEST INFRASTRUCTURE ONLY.
//
//  A plain, unblocked, obviously-correct CPU implementation of the RTM "3D model" time
//  step (arxiv 1310.8232, §2 "3D Stencil Computations": finite differences,
//  10th order in space, 2nd order in time, "five points (cells) in each direction for each
//  dimension"; Algorithm 1 line "forall points: calculate 3D model").
//
//  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
//  leg may load this library.  The product (paper_1310_8232_b200/) never links, imports
//  or executes anything under oracle/, and this file shares no code, header, table or
//  constant generator with the CUDA path.
//
//  What it computes (DESIGN.md §"Readings" R1-R16):
//    U, P : (nz+10)(ny+10)(nx+10) arrays, x fastest, 5-cell zero halo (Dirichlet, R3)
//    Cf[p] = T( (double(v)*double(dt)/double(dx))^2 )                      (a1, R7)
//    for n = 0 .. steps-1:
//       for every interior p (z, y, x ascending):
//          acc = 0
//          for axis in (z, y, x):  for o = -5 .. +5:  acc = acc + c[|o|]*U[p + o*stride]
//          N[p] = (2*U[p] - P[p]) + Cf[p]*acc                                   (a2)
//       for s in registration order: if n < nsamples_s: N[p_s] = N[p_s] + w_s[n] (a3, R4)
//       P <- U, U <- N                                                          (a4)
//  N aliases P because N[p] reads P only at p.
//
//  Compiled with -O2 -ffp-contract=off (no FMA contraction: IEEE-deterministic), OpenMP
//  over z only (per-point arithmetic is independent of the thread count).  FTZ/DAZ is
//  set inside each worker for the fp32 variant (changes only values < 1.2e-38).
//
//  Pins: tests/test_oracle_pins.py (P1-P13 of SURVEY.md §8(c)).  Parity of the wavefield
//  itself is not printed by the paper; every function below is pinned by closed forms,
//  invariants or brute force as listed in DESIGN.md §"Oracle pins".
// =====================================================================================
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>
#include <xmmintrin.h>
#include <pmmintrin.h>

namespace {

constexpr int R = 5;  // stencil radius: "five points (cells) in each direction"

// Wall time of the step loop of the last run() (set-up and copies excluded; SURVEY.md §8(d)
// "time with a steady_clock around the step loop only").  Instrumentation, not arithmetic.
double g_loop_seconds = 0.0;

struct FtzGuard {  // FTZ/DAZ for this thread while alive (fp32 subnormal stalls)
    unsigned int saved;
    explicit FtzGuard(bool on) : saved(_mm_getcsr()) { if (on) _mm_setcsr(saved | 0x8040u); }
    ~FtzGuard() { _mm_setcsr(saved); }
};

template <typename T>
struct Field {
    int nx, ny, nz;
    long sx, sy, sz;  // strides in elements of the padded array
    std::vector<T> a;
    Field(int nx_, int ny_, int nz_) : nx(nx_), ny(ny_), nz(nz_) {
        sx = 1;
        sy = nx + 2 * R;
        sz = (long)(ny + 2 * R) * sy;
        a.assign((size_t)(nz + 2 * R) * sz, T(0));
    }
    long at(int x, int y, int z) const {  // interior coordinates, 0-based
        return (long)(z + R) * sz + (long)(y + R) * sy + (x + R);
    }
};

// The per-point update, written exactly as the definition above.
template <typename T>
inline T update_point(const T* U, const T* P, T cf, const T c[6], long p, long sx, long sy, long sz) {
    T acc = T(0);
    const long strides[3] = {sz, sy, sx};  // axis order (z, y, x) = SPEC's (i, j, k)
    for (int a = 0; a < 3; ++a) {
        for (int o = -R; o <= R; ++o) {
            acc = acc + c[o < 0 ? -o : o] * U[p + o * strides[a]];
        }
    }
    return (T(2) * U[p] - P[p]) + cf * acc;
}

template <typename T, typename VT>
int run(int nx, int ny, int nz, VT dx, VT dt, const T coeffs[6], const VT* v,
        const T* u0, const T* up0, int nsrc, const int* src_xyz, const T* const* samples,
        const int* nsamples, int steps, T* u_out, T* up_out, int nthreads) {
    if (nx < 1 || ny < 1 || nz < 1 || steps < 0 || !v) return -1;
    const bool ftz = sizeof(T) == 4;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    Field<T> U(nx, ny, nz), P(nx, ny, nz), Cf(nx, ny, nz);
    const long sx = U.sx, sy = U.sy, sz = U.sz;
    T c[6];
    for (int k = 0; k < 6; ++k) c[k] = coeffs[k];
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int z = 0; z < nz; ++z) {
        FtzGuard g(ftz);
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const long i = (long)(z * ny + y) * nx + x;
                const long p = U.at(x, y, z);
                // C(p) = (v*dt/dx)^2 in double, rounded once to T (a1; R7)
                const double nu = (double)v[i] * (double)dt / (double)dx;
                Cf.a[p] = (T)(nu * nu);
                U.a[p] = u0 ? u0[i] : T(0);
                P.a[p] = up0 ? up0[i] : T(0);
            }
    }
    std::vector<long> sp(nsrc);
    for (int s = 0; s < nsrc; ++s) {
        const int x = src_xyz[3 * s], y = src_xyz[3 * s + 1], z = src_xyz[3 * s + 2];
        if (x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz) return -2;
        sp[s] = U.at(x, y, z);
    }
    T* Ua = U.a.data();
    T* Pa = P.a.data();
    const T* Ca = Cf.a.data();
    const auto t_loop = std::chrono::steady_clock::now();
    for (int n = 0; n < steps; ++n) {
        T* N = Pa;  // N aliases P
#pragma omp parallel for num_threads(nthreads) schedule(static)
        for (int z = 0; z < nz; ++z) {
            FtzGuard g(ftz);
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const long p = (long)(z + R) * sz + (long)(y + R) * sy + (x + R);
                    N[p] = update_point<T>(Ua, Pa, Ca[p], c, p, sx, sy, sz);
                }
        }
        {
            FtzGuard g(ftz);
            for (int s = 0; s < nsrc; ++s)
                if (n < nsamples[s]) N[sp[s]] = N[sp[s]] + samples[s][n];
        }
        T* t = Pa; Pa = Ua; Ua = t;  // P <- U, U <- N
    }
    g_loop_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_loop).count();
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const long i = (long)(z * ny + y) * nx + x;
                const long p = (long)(z + R) * sz + (long)(y + R) * sy + (x + R);
                if (u_out) u_out[i] = Ua[p];
                if (up_out) up_out[i] = Pa[p];
            }
    return 0;
}

template <typename T>
std::vector<const T*> sample_ptrs(int nsrc, const T* samples, const int* nsamples) {
    std::vector<const T*> ptrs(nsrc);
    long off = 0;
    for (int s = 0; s < nsrc; ++s) { ptrs[s] = samples + off; off += nsamples[s]; }
    return ptrs;
}

}  // namespace

extern "C" {

// Full run in fp32 (the parity oracle).  Arrays are unpadded interior arrays,
// index (z*ny + y)*nx + x.  u0/up0 may be NULL (zero initial conditions).
// Sources: src_xyz[3*s..3*s+2] = (x, y, z); samples are concatenated per source with
// lengths nsamples[s].  u_out receives u^steps, up_out (may be NULL) u^(steps-1).
// Returns 0, -1 on bad sizes, -2 on a source outside the interior.
int oracle_run_f32(int nx, int ny, int nz, float dx, float dt, const float coeffs[6],
                   const float* v, const float* u0, const float* up0, int nsrc,
                   const int* src_xyz, const float* samples, const int* nsamples, int steps,
                   float* u_out, float* up_out, int nthreads) {
    auto ptrs = sample_ptrs<float>(nsrc, samples, nsamples);
    return run<float, float>(nx, ny, nz, dx, dt, coeffs, v, u0, up0, nsrc, src_xyz, ptrs.data(),
                             nsamples, steps, u_out, up_out, nthreads);
}

// The same definition in fp64 throughout (v, dx, dt and coefficients in double).
int oracle_run_f64(int nx, int ny, int nz, double dx, double dt, const double coeffs[6],
                   const double* v, const double* u0, const double* up0, int nsrc,
                   const int* src_xyz, const double* samples, const int* nsamples, int steps,
                   double* u_out, double* up_out, int nthreads) {
    auto ptrs = sample_ptrs<double>(nsrc, samples, nsamples);
    return run<double, double>(nx, ny, nz, dx, dt, coeffs, v, u0, up0, nsrc, src_xyz,
                               ptrs.data(), nsamples, steps, u_out, up_out, nthreads);
}

// One fp32 step evaluated only at the listed interior points (for sampled parity checks
// at full config sizes, where a whole-grid oracle step is too slow).  Same definition:
// out[k] = (2u - up) + C*acc at point pts[3k..3k+2] = (x, y, z); neighbours outside the
// interior read 0 (the zero halo).  No source term (callers add w themselves if needed).
int oracle_points_f32(int nx, int ny, int nz, float dx, float dt, const float coeffs[6],
                      const float* v, const float* u, const float* up, long npts,
                      const int* pts, float* out) {
    if (nx < 1 || ny < 1 || nz < 1) return -1;
    FtzGuard g(true);
    const long sxy = (long)nx * ny;
    for (long k = 0; k < npts; ++k) {
        const int x = pts[3 * k], y = pts[3 * k + 1], z = pts[3 * k + 2];
        if (x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz) return -2;
        auto U = [&](int xx, int yy, int zz) -> float {
            if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz) return 0.0f;
            return u[(long)zz * sxy + (long)yy * nx + xx];
        };
        float acc = 0.0f;
        for (int o = -R; o <= R; ++o) acc = acc + coeffs[o < 0 ? -o : o] * U(x, y, z + o);
        for (int o = -R; o <= R; ++o) acc = acc + coeffs[o < 0 ? -o : o] * U(x, y + o, z);
        for (int o = -R; o <= R; ++o) acc = acc + coeffs[o < 0 ? -o : o] * U(x + o, y, z);
        const long i = (long)z * sxy + (long)y * nx + x;
        const double nu = (double)v[i] * (double)dt / (double)dx;
        const float cf = (float)(nu * nu);
        out[k] = (2.0f * u[i] - up[i]) + cf * acc;
    }
    return 0;
}

// One fp32 step of a z-slab with EXPLICIT z-halo planes (the CPU slab simulator used to
// check domain decomposition, SURVEY.md §4 "CPU slab simulator").  U and P hold nzl+10
// planes of nx*ny (planes 0..4 and nzl+5..nzl+9 are the z-halo, owned planes at 5..nzl+4);
// the x/y halo is zero.  Writes N into P's owned planes (N aliases P).  C is nzl planes,
// already C(p) (computed by the caller with the same formula as oracle_run_f32).
int oracle_slab_step_f32(int nx, int ny, int nzl, const float coeffs[6], const float* C,
                         const float* U, float* P, int nthreads) {
    if (nx < 1 || ny < 1 || nzl < 1) return -1;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    const long sxy = (long)nx * ny;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int zl = 0; zl < nzl; ++zl) {
        FtzGuard g(true);
        const int zb = zl + R;  // buffer plane
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                auto Uv = [&](int xx, int yy, int zz) -> float {
                    if (xx < 0 || xx >= nx || yy < 0 || yy >= ny) return 0.0f;
                    return U[(long)zz * sxy + (long)yy * nx + xx];
                };
                float acc = 0.0f;
                for (int o = -R; o <= R; ++o) acc = acc + coeffs[o < 0 ? -o : o] * Uv(x, y, zb + o);
                for (int o = -R; o <= R; ++o) acc = acc + coeffs[o < 0 ? -o : o] * Uv(x, y + o, zb);
                for (int o = -R; o <= R; ++o) acc = acc + coeffs[o < 0 ? -o : o] * Uv(x + o, y, zb);
                const long p = (long)zb * sxy + (long)y * nx + x;
                P[p] = (2.0f * U[p] - P[p]) + C[(long)zl * sxy + (long)y * nx + x] * acc;
            }
    }
    return 0;
}

// C(p) = fp32((v*dt/dx)^2) computed in double (a1), for the slab simulator.
int oracle_cfield_f32(long n, float dx, float dt, const float* v, float* C) {
    for (long i = 0; i < n; ++i) {
        const double nu = (double)v[i] * (double)dt / (double)dx;
        C[i] = (float)(nu * nu);
    }
    return 0;
}

int oracle_max_threads(void) { return omp_get_max_threads(); }

// Seconds spent in the step loop of the last oracle_run_f32/f64 call (bench timing only).
double oracle_last_loop_seconds(void) { return g_loop_seconds; }

}  // extern "C"
