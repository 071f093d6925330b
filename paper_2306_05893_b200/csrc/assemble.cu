// Fused corotational assembly into a fixed CSR pattern.
//
// Replaces, on the device, the per-step work of
//   BackwardEulerIntegrator.assemble_system     integrator.py:145-169
//   corotational_forces_and_stiffness           models.py:200-238
//   polar_rotations                             models.py:174-189
//   MatrixAssembler.finish -> compress          assembly.py:407-419, 332-343
//
// Two launches, no atomics, fixed summation order (the block and node gathers
// share one launch, gather_kernel):
//   1. elem_kernel   one thread per tetrahedron: F = sum_a x_a g_a^T, Newton
//                    polar R <- (R + R^-T)/2, rotated gradients g^_a = R g_a,
//                    f_e = R Ke (R^T x - x0) and (K v)_e = R Ke R^T v in
//                    stress form (no 12x12 Ke is ever read: 104 B of rest data
//                    per tet instead of 1,152 B).
//   2. gather_kernel (block part) one thread per 3x3 node block of the CSR pattern: sums
//                    cm*mass (diagonal blocks) then ck*(R Ke R^T)_ab over the
//                    contributing elements in ascending element order -- the
//                    ascending-triplet order np.bincount uses
//                    (assembly.py:341), so slot sums follow the reference's
//                    association exactly.  Block entry (i,j) of element e:
//                    V (lam g^_a,i g^_b,j + mu g^_a,j g^_b,i + mu (g_a.g_b) d_ij)
//   3. gather_kernel (node part) one thread per node: f_int and K v gathered over incident
//                    elements in ascending order (np.bincount order,
//                    models.py:192-193), then
//                    b = f_ext - f_int - (h+beta) K v - alpha M v, b[pinned]=0
//                    (integrator.py:158-162), every operation rounded as NumPy
//                    rounds it.
//
// Material laws (tsb_asm_coeffs.law): corotational (above), linear (R := I)
// and St-Venant-Kirchhoff (stvk_forces_and_stiffness, models.py:241-287).
// For StVK the element pass stores h_a = F g_a in place of the rotated
// gradients plus F F^T and S (second Piola-Kirchhoff stress) in an auxiliary
// [m][12] region after the [m][36] scratch; f_e = V F S g_a and, in stress
// form, (K v)_a = V(lam (sum_b h_b.v_b) h_a + mu W h_a + mu F F^T Hv g_a
// + Hv S g_a) with W = sum_b h_b v_b^T, Hv = sum_b v_b g_b^T -- the 12x12
// element tangent is never formed.  The block pass evaluates
// K_ab = V(lam h_a h_b^T + mu h_b h_a^T + mu (g_a.g_b) F F^T + (g_a^T S g_b) I)
// in the reference's term order.
#include <cstdlib>

#include "tsb_common.cuh"

namespace tsb {

constexpr int kWork = 36;  // per-element scratch: g^[12], f_e[12], (Kv)_e[12]
constexpr int kAux = 12;   // StVK: F F^T (xx xy xz yy yz zz), S (same order), after m * kWork

__device__ __forceinline__ bool finite3(double a, double b, double c) {
    return isfinite(a) && isfinite(b) && isfinite(c);
}

// R <- (R + R^{-T}) / 2 until max |dR| < tol (models.py:174-189), per element.
__device__ __forceinline__ void polar(const double F[9], double R[9]) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = F[k];
    for (int it = 0; it < 50; ++it) {
        // cofactor matrix C: inv(R)^T = C / det
        double c00 = R[4] * R[8] - R[5] * R[7];
        double c01 = R[5] * R[6] - R[3] * R[8];
        double c02 = R[3] * R[7] - R[4] * R[6];
        double c10 = R[2] * R[7] - R[1] * R[8];
        double c11 = R[0] * R[8] - R[2] * R[6];
        double c12 = R[1] * R[6] - R[0] * R[7];
        double c20 = R[1] * R[5] - R[2] * R[4];
        double c21 = R[2] * R[3] - R[0] * R[5];
        double c22 = R[0] * R[4] - R[1] * R[3];
        double det = R[0] * c00 + R[1] * c01 + R[2] * c02;
        double id = 1.0 / det;
        double C[9] = {c00, c01, c02, c10, c11, c12, c20, c21, c22};
        double delta = 0.0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            double nr = 0.5 * (R[k] + C[k] * id);
            delta = fmax(delta, fabs(nr - R[k]));
            R[k] = nr;
        }
        if (delta < 1e-12) break;
    }
}

// (Ke u)_a = V sigma g_a with sigma = lam tr(H) I + mu (H + H^T), H = sum_b u_b g_b^T.
__device__ __forceinline__ void ke_apply(const double u[12], const double g[12], double V,
                                         double lam, double mu, double out[12]) {
    double H[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            H[3 * i + j] = u[i] * g[j] + u[3 + i] * g[3 + j] + u[6 + i] * g[6 + j] + u[9 + i] * g[9 + j];
    const double tr = H[0] + H[4] + H[8];
    double S[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) S[3 * i + j] = mu * (H[3 * i + j] + H[3 * j + i]) + (i == j ? lam * tr : 0.0);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            out[3 * a + i] = V * (S[3 * i] * g[3 * a] + S[3 * i + 1] * g[3 * a + 1] + S[3 * i + 2] * g[3 * a + 2]);
}

// St-Venant-Kirchhoff element pass (models.py:258-285), see the header.
__device__ __forceinline__ void stvk_element(int64_t e, int64_t m, const double g[12], const double xe[12],
                                             const double ve[12], double V, double lam, double mu,
                                             double *__restrict__ work) {
    double F[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            F[3 * i + j] = xe[i] * g[j] + xe[3 + i] * g[3 + j] + xe[6 + i] * g[6 + j] + xe[9 + i] * g[9 + j];
    double S[9], FFt[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            S[3 * i + j] = 0.5 * ((F[i] * F[j] + F[3 + i] * F[3 + j] + F[6 + i] * F[6 + j]) - (i == j ? 1.0 : 0.0));
            FFt[3 * i + j] = F[3 * i] * F[3 * j] + F[3 * i + 1] * F[3 * j + 1] + F[3 * i + 2] * F[3 * j + 2];
        }
    const double trg = S[0] + S[4] + S[8];
#pragma unroll
    for (int k = 0; k < 9; ++k) S[k] = 2.0 * mu * S[k] + (k % 4 == 0 ? lam * trg : 0.0);
    double FS[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) FS[3 * i + j] = F[3 * i] * S[j] + F[3 * i + 1] * S[3 + j] + F[3 * i + 2] * S[6 + j];
    double h[12], t[12];
    double s1 = 0.0, W[9], Hv[9];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            h[3 * a + i] = F[3 * i] * g[3 * a] + F[3 * i + 1] * g[3 * a + 1] + F[3 * i + 2] * g[3 * a + 2];
            t[3 * a + i] = V * (FS[3 * i] * g[3 * a] + FS[3 * i + 1] * g[3 * a + 1] + FS[3 * i + 2] * g[3 * a + 2]);
        }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            W[3 * i + k] = h[i] * ve[k] + h[3 + i] * ve[3 + k] + h[6 + i] * ve[6 + k] + h[9 + i] * ve[9 + k];
            Hv[3 * i + k] = ve[i] * g[k] + ve[3 + i] * g[3 + k] + ve[6 + i] * g[6 + k] + ve[9 + i] * g[9 + k];
        }
#pragma unroll
    for (int a = 0; a < 12; ++a) s1 += h[a] * ve[a];
    double2 *out = reinterpret_cast<double2 *>(work + e * kWork);
#pragma unroll
    for (int k = 0; k < 6; ++k) out[k] = make_double2(h[2 * k], h[2 * k + 1]);
#pragma unroll
    for (int k = 0; k < 6; ++k) out[6 + k] = make_double2(t[2 * k], t[2 * k + 1]);
    // M1 = mu FF^T Hv + Hv S, so the last two terms are M1 g_a
    double M1[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            M1[3 * i + j] = mu * (FFt[3 * i] * Hv[j] + FFt[3 * i + 1] * Hv[3 + j] + FFt[3 * i + 2] * Hv[6 + j]) +
                            (Hv[3 * i] * S[j] + Hv[3 * i + 1] * S[3 + j] + Hv[3 * i + 2] * S[6 + j]);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            t[3 * a + i] = V * (lam * s1 * h[3 * a + i] +
                                mu * (W[3 * i] * h[3 * a] + W[3 * i + 1] * h[3 * a + 1] + W[3 * i + 2] * h[3 * a + 2]) +
                                (M1[3 * i] * g[3 * a] + M1[3 * i + 1] * g[3 * a + 1] + M1[3 * i + 2] * g[3 * a + 2]));
#pragma unroll
    for (int k = 0; k < 6; ++k) out[12 + k] = make_double2(t[2 * k], t[2 * k + 1]);
    double2 *aux = reinterpret_cast<double2 *>(work + m * kWork + e * kAux);
    aux[0] = make_double2(FFt[0], FFt[1]);
    aux[1] = make_double2(FFt[2], FFt[4]);
    aux[2] = make_double2(FFt[5], FFt[8]);
    aux[3] = make_double2(S[0], S[1]);
    aux[4] = make_double2(S[2], S[4]);
    aux[5] = make_double2(S[5], S[8]);
}

__global__ void __launch_bounds__(128, 4)
elem_kernel(int64_t m, const int32_t *__restrict__ conn, const double *__restrict__ grads,
            const double *__restrict__ vol, const double *__restrict__ rest,
            const double *__restrict__ x, const double *__restrict__ v, double lam, double mu,
            int law, double *__restrict__ work, int32_t *__restrict__ flags) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m) return;
    int nd[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) nd[a] = __ldg(conn + a * m + e);
    double g[12], xe[12], ve[12], x0[12];
    const double2 *g2 = reinterpret_cast<const double2 *>(grads + e * 12);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        double2 t = __ldg(g2 + k);
        g[2 * k] = t.x;
        g[2 * k + 1] = t.y;
    }
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            xe[3 * a + i] = __ldg(x + 3 * nd[a] + i);
            ve[3 * a + i] = v ? __ldg(v + 3 * nd[a] + i) : 0.0;
            x0[3 * a + i] = __ldg(rest + 3 * nd[a] + i);
        }
        ok = ok && finite3(xe[3 * a], xe[3 * a + 1], xe[3 * a + 2]);
    }
    if (!ok) atomicOr(flags, 1);
    const double V = __ldg(vol + e);
    if (law == TSB_LAW_STVK) {
        stvk_element(e, m, g, xe, ve, V, lam, mu, work);
        return;
    }

    double R[9];
    if (law == TSB_LAW_LINEAR) {
#pragma unroll
        for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? 1.0 : 0.0;
    } else {
        double F[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                F[3 * i + j] = xe[i] * g[j] + xe[3 + i] * g[3 + j] + xe[6 + i] * g[6 + j] + xe[9 + i] * g[9 + j];
        polar(F, R);
    }

    // u_a = R^T x_a - x0_a  (models.py:227, same order as the reference)
    double u[12], w[12], t[12];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            u[3 * a + i] = (R[i] * xe[3 * a] + R[3 + i] * xe[3 * a + 1] + R[6 + i] * xe[3 * a + 2]) - x0[3 * a + i];
            w[3 * a + i] = R[i] * ve[3 * a] + R[3 + i] * ve[3 * a + 1] + R[6 + i] * ve[3 * a + 2];
        }
    double2 *out = reinterpret_cast<double2 *>(work + e * kWork);
    // rotated gradients
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            t[3 * a + i] = R[3 * i] * g[3 * a] + R[3 * i + 1] * g[3 * a + 1] + R[3 * i + 2] * g[3 * a + 2];
#pragma unroll
    for (int k = 0; k < 6; ++k) out[k] = make_double2(t[2 * k], t[2 * k + 1]);
    // f_e = R (Ke u)
    double ku[12];
    ke_apply(u, g, V, lam, mu, ku);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            t[3 * a + i] = R[3 * i] * ku[3 * a] + R[3 * i + 1] * ku[3 * a + 1] + R[3 * i + 2] * ku[3 * a + 2];
#pragma unroll
    for (int k = 0; k < 6; ++k) out[6 + k] = make_double2(t[2 * k], t[2 * k + 1]);
    // (K v)_e = R (Ke (R^T v))
    ke_apply(w, g, V, lam, mu, ku);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            t[3 * a + i] = R[3 * i] * ku[3 * a] + R[3 * i + 1] * ku[3 * a + 1] + R[3 * i + 2] * ku[3 * a + 2];
#pragma unroll
    for (int k = 0; k < 6; ++k) out[12 + k] = make_double2(t[2 * k], t[2 * k + 1]);
}

// Rotated element block entry (R Ke_ab R^T)_ij.
__device__ __forceinline__ void rot_block(const double *ga, const double *gb, double G, double V,
                                          double lam, double mu, double k[9]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            k[3 * i + j] = V * (lam * ga[i] * gb[j] + mu * ga[j] * gb[i] + (i == j ? mu * G : 0.0));
}

// StVK element block entry (models.py:272-279, same term order):
// V (((lam h_a,i h_b,k + mu h_a,k h_b,i) + mu (G fft_ik)) + gsg d_ik).
__device__ __forceinline__ void stvk_block(const double *ha, const double *hb, const double *ra,
                                           const double *rb, const double aux[12], double V, double lam,
                                           double mu, double k[9]) {
    const double G = ra[0] * rb[0] + ra[1] * rb[1] + ra[2] * rb[2];
    const double S[9] = {aux[6], aux[7], aux[8], aux[7], aux[9], aux[10], aux[8], aux[10], aux[11]};
    const double P[9] = {aux[0], aux[1], aux[2], aux[1], aux[3], aux[4], aux[2], aux[4], aux[5]};
    double sb[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) sb[j] = S[3 * j] * rb[0] + S[3 * j + 1] * rb[1] + S[3 * j + 2] * rb[2];
    const double gsg = ra[0] * sb[0] + ra[1] * sb[1] + ra[2] * sb[2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double v = add(add(mul(lam, mul(ha[i], hb[j])), mul(mu, mul(ha[j], hb[i]))), mul(mu, mul(G, P[3 * i + j])));
            if (i == j) v = add(v, gsg);
            k[3 * i + j] = mul(v, V);
        }
}

__device__ __forceinline__ void load_aux(const double *__restrict__ work, int64_t m, int64_t e, double aux[12]) {
    const double2 *p = reinterpret_cast<const double2 *>(work + m * kWork + e * kAux);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 t = __ldg(p + k);
        aux[2 * k] = t.x;
        aux[2 * k + 1] = t.y;
    }
}

// slot of the symmetric pair (a, b) in a tet's 10 rest-gradient products
__device__ __forceinline__ int gab_slot(int a, int b) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo * 4 - lo * (lo - 1) / 2 + (hi - lo);  // (0,0..3) 0..3, (1,1..3) 4..6, (2,2..3) 7..8, (3,3) 9
}

// gab[e][slot(a, b)] = g_a . g_b (plan setup; the same expression the block
// gather evaluated per contribution)
__global__ void gab_kernel(int64_t m, const double *__restrict__ grads, double *__restrict__ gab) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m) return;
    double g[12];
#pragma unroll
    for (int t = 0; t < 12; ++t) g[t] = grads[e * 12 + t];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a; b < 4; ++b)
            gab[e * 10 + gab_slot(a, b)] = g[3 * a] * g[3 * b] + g[3 * a + 1] * g[3 * b + 1] + g[3 * a + 2] * g[3 * b + 2];
}

template <bool STVK, int U>
__device__ __forceinline__ void block_body(int64_t bi, int64_t nb, int64_t m, const int4 *__restrict__ blk,
                                           const int2 *__restrict__ mirror,
                                           const int32_t *__restrict__ list, const double *__restrict__ work,
                                           const double *__restrict__ grads, const double *__restrict__ gab,
                                           const double *__restrict__ vol,
                                           const double *__restrict__ share, double lam, double mu, double cm,
                                           double ck, double *__restrict__ values) {
    if (bi >= nb) return;
    const int4 info = __ldg(blk + bi);  // slot0, rowlen, begin, end
    double acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.0;
    const int c0 = __ldg(list + info.z);
    const bool diag = ((c0 >> 2) & 3) == (c0 & 3);
    if (diag) {
        // mass triplets first (indices < 12 m), ascending element
        for (int k = info.z; k < info.w; ++k) {
            const double mv = mul(cm, __ldg(share + (__ldg(list + k) >> 4)));
            acc[0] = add(acc[0], mv);
            acc[4] = add(acc[4], mv);
            acc[8] = add(acc[8], mv);
        }
    }
    // contributions in ascending element order; the loads of U contributions
    // are issued before their (ordered) accumulation
    // U contributions' loads in flight per thread (template)
    for (int k0 = info.z; k0 < info.w; k0 += U) {
        double ga[U][3], gb[U][3], G[U], V[U];
        double ra[U][3], rb[U][3], aux[STVK ? U : 1][12];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u < info.w ? k0 + u : info.w - 1;
            const int c = __ldg(list + k);
            const int64_t e = c >> 4;
            const int a = (c >> 2) & 3, b = c & 3;
            const double *we = work + e * kWork;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                ga[u][i] = __ldg(we + 3 * a + i);
                gb[u][i] = __ldg(we + 3 * b + i);
            }
            if constexpr (STVK) {
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    ra[u][i] = __ldg(grads + e * 12 + 3 * a + i);
                    rb[u][i] = __ldg(grads + e * 12 + 3 * b + i);
                }
                load_aux(work, m, e, aux[u]);
                G[u] = 0.0;
            } else {  // g_a . g_b of the rest gradients, tabulated once per plan
                G[u] = __ldg(gab + e * 10 + gab_slot(a, b));
            }
            V[u] = __ldg(vol + e);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u >= info.w) break;
            double kb[9];
            if constexpr (STVK)
                stvk_block(ga[u], gb[u], ra[u], rb[u], aux[u], V[u], lam, mu, kb);
            else
                rot_block(ga[u], gb[u], G[u], V[u], lam, mu, kb);
#pragma unroll
            for (int q = 0; q < 9; ++q) acc[q] = add(acc[q], mul(ck, kb[q]));
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) values[info.x + i * info.y + j] = acc[3 * i + j];
    if (mirror != nullptr) {  // K_ba = K_ab^T (the element blocks are symmetric): block (J, I) from (I, J)
        const int2 mb = __ldg(mirror + bi);
        if (mb.x >= 0) {
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) values[mb.x + j * mb.y + i] = acc[3 * i + j];
        }
    }
}

__device__ __forceinline__ void node_body(int64_t I, int64_t N, const int32_t *__restrict__ node_ptr,
                                          const int32_t *__restrict__ node_list, const double *__restrict__ work,
                                          const double *__restrict__ x, const double *__restrict__ v,
                                          const double *__restrict__ fext_state, const double *__restrict__ gravity,
                                          const double *__restrict__ mass_diag, const uint8_t *__restrict__ fixed,
                                          double hb, double alpha, double *__restrict__ f_int,
                                          double *__restrict__ kv, double *__restrict__ b,
                                          double *__restrict__ f_ext, int32_t *__restrict__ flags) {
    if (I >= N) return;
    if (!finite3(x[3 * I], x[3 * I + 1], x[3 * I + 2])) atomicOr(flags, 1);
    double f[3] = {0.0, 0.0, 0.0}, k[3] = {0.0, 0.0, 0.0};
    const int lo = __ldg(node_ptr + I), hi = __ldg(node_ptr + I + 1);
    // incident elements in ascending order (np.bincount's order); the loads of
    // U incidences are issued before their ordered accumulation
    constexpr int U = 4;
    for (int q0 = lo; q0 < hi; q0 += U) {
        double fv[U][3], kv_[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = q0 + u < hi ? q0 + u : hi - 1;
            const int c = __ldg(node_list + q);
            const double *we = work + (int64_t)(c >> 2) * kWork + 3 * (c & 3);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                fv[u][i] = __ldg(we + 12 + i);
                kv_[u][i] = __ldg(we + 24 + i);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (q0 + u >= hi) break;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                f[i] = add(f[i], fv[u][i]);
                k[i] = add(k[i], kv_[u][i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int64_t d = 3 * I + i;
        f_int[d] = f[i];
        kv[d] = k[i];
        if (b != nullptr) {
            const double fe = add(fext_state[d], gravity[d]);
            double r = sub(sub(fe, f[i]), mul(hb, k[i]));
            if (alpha != 0.0) r = sub(r, mul(alpha, mul(mass_diag[d], v[d])));
            if (fixed[d]) r = 0.0;
            b[d] = r;
            if (f_ext != nullptr) f_ext[d] = fe;
        }
    }
}

// One launch for both gathers: node CTAs gather the nodes' f_int / K v / rhs
// (thread per node), block CTAs sum the 3x3 blocks (thread per block); the two
// are independent, so the small node gather overlaps the block gather instead
// of running after it.
template <bool STVK, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
gather_kernel(int64_t nbc, int64_t nb, int64_t m, const int4 *__restrict__ blk, const int2 *__restrict__ mirror,
              const int32_t *__restrict__ list,
              const double *__restrict__ work, const double *__restrict__ grads, const double *__restrict__ gab,
              const double *__restrict__ vol,
              const double *__restrict__ share, double lam, double mu, double cm, double ck,
              double *__restrict__ values, int64_t N, const int32_t *__restrict__ node_ptr,
              const int32_t *__restrict__ node_list, const double *__restrict__ x, const double *__restrict__ v,
              const double *__restrict__ fext_state, const double *__restrict__ gravity,
              const double *__restrict__ mass_diag, const uint8_t *__restrict__ fixed, double hb, double alpha,
              double *__restrict__ f_int, double *__restrict__ kv, double *__restrict__ b,
              double *__restrict__ f_ext, int32_t *__restrict__ flags) {
    // CTA order: each node CTA is followed by the r block CTAs covering about
    // the same node rows (blocks are in node-row order, ~r blocks per node), so
    // an element's scratch row is read by its nodes and its blocks while it is
    // still in L2; leftover block CTAs come last
    const int64_t nnc = (N + blockDim.x - 1) / blockDim.x;
    const int64_t r = nnc > 0 ? nbc / nnc : 0;
    const int64_t bx = blockIdx.x;
    int64_t node_cta = -1, blk_cta;
    if (bx < nnc * (r + 1)) {
        const int64_t g = bx / (r + 1), o = bx % (r + 1);
        if (o == 0) node_cta = g;
        blk_cta = g * r + (o - 1);
    } else {
        blk_cta = nnc * r + (bx - nnc * (r + 1));
    }
    if (node_cta >= 0)
        node_body(node_cta * (int64_t)blockDim.x + threadIdx.x, N, node_ptr, node_list, work, x, v, fext_state,
                  gravity, mass_diag, fixed, hb, alpha, f_int, kv, b, f_ext, flags);
    else
        block_body<STVK, U>(blk_cta * (int64_t)blockDim.x + threadIdx.x, nb, m, blk, mirror, list, work, grads, gab,
                            vol, share, lam, mu, cm, ck, values);
}

__global__ void __launch_bounds__(128)
kblock_kernel(int64_t m, const double *__restrict__ work, const double *__restrict__ grads,
              const double *__restrict__ vol, double lam, double mu, int law, double *__restrict__ out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m) return;
    const double *we = work + e * kWork;
    const double V = vol[e];
    double aux[12];
    if (law == TSB_LAW_STVK) load_aux(work, m, e, aux);
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            const double *ra = grads + e * 12 + 3 * a, *rb = grads + e * 12 + 3 * b;
            double kb[9];
            if (law == TSB_LAW_STVK)
                stvk_block(we + 3 * a, we + 3 * b, ra, rb, aux, V, lam, mu, kb);
            else
                rot_block(we + 3 * a, we + 3 * b, ra[0] * rb[0] + ra[1] * rb[1] + ra[2] * rb[2], V, lam, mu, kb);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) out[e * 144 + (3 * a + i) * 12 + 3 * b + j] = kb[3 * i + j];
        }
}

// Kinematic update of one implicit step (integrator.py:192-208):
// non-finite accel -> flag (StepError); accel[pinned] = 0; v' = v + h a;
// x' = x + h v'; pinned DOFs keep v and x.
__global__ void advance_kernel(int64_t n, const double *__restrict__ acc, const double *__restrict__ v,
                               const double *__restrict__ x, const uint8_t *__restrict__ fixed, double h,
                               double *__restrict__ acc_out, double *__restrict__ v_out,
                               double *__restrict__ x_out, int32_t *__restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double a = acc[i];
        if (!isfinite(a)) atomicOr(flags + 1, 1);
        const bool pin = fixed[i] != 0;
        if (pin) a = 0.0;
        double vv = add(v[i], mul(h, a));
        double xx = add(x[i], mul(h, vv));
        if (pin) {
            vv = v[i];
            xx = x[i];
        }
        acc_out[i] = a;
        v_out[i] = vv;
        x_out[i] = xx;
    }
}

__global__ void set_ones_kernel(int64_t n, const int32_t *__restrict__ slots, double *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[slots[i]] = 1.0;
}

static inline int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    return (int)(g > 0 ? g : 1);
}

void launch_elem(const tsb_asm_plan *p, const tsb_asm_coeffs *c, const double *x, const double *v,
                 cudaStream_t s) {
    if (p->n_elems <= 0) return;
    elem_kernel<<<grid_for(p->n_elems, 128), 128, 0, s>>>(p->n_elems, p->d_conn, p->d_grads, p->d_vol,
                                                          p->d_rest, x, v, c->lam, c->mu, c->law,
                                                          p->d_work, p->d_flags);
    TSB_LAUNCHED();
}

}  // namespace tsb

extern "C" int tsb_assemble_corot(const tsb_asm_plan *p, const tsb_asm_coeffs *c, const double *d_x,
                                  const double *d_v, const double *d_f_ext_state, double *d_values,
                                  double *d_b, double *d_f_int, double *d_kv, double *d_f_ext,
                                  void *stream) {
    using namespace tsb;
    return guard([&] {
        if (p == nullptr || c == nullptr) throw Error(TSB_E_ARG, "null plan/coeffs");
        if (c->law < TSB_LAW_COROTATIONAL || c->law > TSB_LAW_STVK) throw Error(TSB_E_ARG, "unknown material law");
        cudaStream_t s = as_stream(stream);
        TSB_CUDA(cudaMemsetAsync(p->d_flags, 0, 4 * sizeof(int32_t), s));  // status words of this pass
        launch_elem(p, c, d_x, d_v, s);
        const bool mat = c->want_matrix && d_values != nullptr;
        const int64_t nbc = mat && p->n_blocks > 0 ? grid_for(p->n_blocks, 256) : 0;
        const int64_t nnc = p->n_nodes > 0 ? grid_for(p->n_nodes, 256) : 0;
        if (nbc + nnc > 0) {
            // occupancy vs loads in flight per thread (TSB_GATHER_VARIANT, measured in tools/asm_bench.py)
            static const int variant = getenv("TSB_GATHER_VARIANT") ? atoi(getenv("TSB_GATHER_VARIANT")) : 0;
            auto kern = c->law == TSB_LAW_STVK ? gather_kernel<true, 4, 1> : gather_kernel<false, 4, 1>;
            if (c->law != TSB_LAW_STVK) {
                if (variant == 1) kern = gather_kernel<false, 2, 6>;
                else if (variant == 2) kern = gather_kernel<false, 4, 4>;
                else if (variant == 3) kern = gather_kernel<false, 2, 4>;
                else if (variant == 4) kern = gather_kernel<false, 1, 8>;
            }
            kern<<<(unsigned)(nbc + nnc), 256, 0, s>>>(
                nbc, p->n_blocks, p->n_elems, reinterpret_cast<const int4 *>(p->d_blk),
                reinterpret_cast<const int2 *>(p->d_blk_mirror), p->d_blk_list, p->d_work,
                p->d_grads, p->d_gab, p->d_vol, p->d_mass_share, c->lam, c->mu, c->cm, c->ck, d_values, p->n_nodes,
                p->d_node_ptr, p->d_node_list, d_x, d_v, d_f_ext_state, p->d_gravity, p->d_mass_diag,
                p->d_fixed_dof, c->h + c->rayleigh_stiffness, c->rayleigh_mass, d_f_int, d_kv, d_b, d_f_ext,
                p->d_flags);
            TSB_LAUNCHED();
        }
        if (mat && p->n_fixed_slots > 0) {
            set_ones_kernel<<<grid_for(p->n_fixed_slots, 256), 256, 0, s>>>(p->n_fixed_slots, p->d_fixed_slots,
                                                                            d_values);
            TSB_LAUNCHED();
        }
    });
}

extern "C" int tsb_element_blocks(const tsb_asm_plan *p, const tsb_asm_coeffs *c, const double *d_x,
                                  double *d_kblocks, void *stream) {
    using namespace tsb;
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        launch_elem(p, c, d_x, nullptr, s);
        if (p->n_elems > 0) {
            kblock_kernel<<<grid_for(p->n_elems, 128), 128, 0, s>>>(p->n_elems, p->d_work, p->d_grads,
                                                                    p->d_vol, c->lam, c->mu, c->law, d_kblocks);
            TSB_LAUNCHED();
        }
    });
}

extern "C" int tsb_advance(int64_t n_dof, const double *d_accel, const double *d_v, const double *d_x,
                           const uint8_t *d_fixed_dof, double h, double *d_acc_out, double *d_v_out,
                           double *d_x_out, int32_t *d_flags, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (n_dof <= 0) return;
        int g = grid_for(n_dof, 256);
        if (g > kNumSM * 8) g = kNumSM * 8;
        advance_kernel<<<g, 256, 0, as_stream(stream)>>>(n_dof, d_accel, d_v, d_x, d_fixed_dof, h,
                                                         d_acc_out, d_v_out, d_x_out, d_flags);
        TSB_LAUNCHED();
    });
}

// Plan setup: the rest-gradient products g_a . g_b per tet into d_gab
// ([m][10]), read by the block gather instead of the two gradient rows.
extern "C" int tsb_assembly_setup(const tsb_asm_plan *p, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (p == nullptr || p->d_gab == nullptr) throw Error(TSB_E_ARG, "plan without a g_a.g_b table");
        if (p->n_elems <= 0) return;
        gab_kernel<<<grid_for(p->n_elems, 128), 128, 0, as_stream(stream)>>>(p->n_elems, p->d_grads,
                                                                             const_cast<double *>(p->d_gab));
        TSB_LAUNCHED();
    });
}
