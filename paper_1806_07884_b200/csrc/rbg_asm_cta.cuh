// rbg_asm_cta.cuh -- the CTA-cooperative assembly kernel (K3), included by
// rbg_asm.cuh.  Same arithmetic and the same two-level layout as the
// one-warp kernel (super-tiles of sub-tiles, slot-map flush), organised for
// occupancy instead of one warp owning everything:
//
//   * a CTA of 4 warps owns a super-tile: one shared accumulator (dense upper
//     triangle of the super-tile's centre pairs), one staged slot map;
//   * per sub-tile and chunk of up to 8 four-point k-steps:
//       phi phase  -- warp w evaluates the DMMA fragments of the row blocks
//                     I = w (mod 4) (phi_at: exact inclusion, the reference's
//                     t and u) into a shared fragment buffer, and keeps
//                     A^T h / hit counts of those rows in registers;
//       SYRK phase -- the NB(NB+1)/2 upper 8x8 blocks are split into four
//                     contiguous ranges fixed at compile time; warp w loads the
//                     NB fragments of each k-step once and runs its DMMAs
//                     (m8n8k4 f64) into register tiles that persist across
//                     chunks;
//   * fold -- each warp adds its blocks into the shared accumulator (the blocks
//     of one sub-tile are disjoint, sub-tiles are separated by a barrier, so
//     plain read-modify-write is race free);
//   * flush at super-tile end: one fp64 global reduction per nonzero pair.
// phi is still evaluated once per (point, centre) pair; a warp needs at most
// 2 x 9 accumulator doubles, so registers stay low and 4 CTAs (16 warps) fit
// an SM where the one-warp kernel fits 8 warps.
#pragma once

namespace rbg {
namespace {

constexpr int CW = 4;        // warps per CTA
constexpr int CT = CW * 32;  // threads per CTA
constexpr int CKS = 8;       // k-steps per fragment chunk
constexpr int CNB = 8;       // largest sub-tile handled: 8 blocks = 64 centres

struct CGeom {
    BlobLayout B;
    int lsb, lsub_cap, map_staged;
    uint32_t blob, map, sp, acc, rhs, hits, gath, phi, misc, region;
};

CGeom plan_cgeom(int dim, int lsb, int lsub_cap, int sd, int stage_map) {
    CGeom g{};
    g.B = blob_layout(dim, lsb, sd, lsub_cap);
    g.lsb = lsb;
    g.lsub_cap = lsub_cap;
    g.map_staged = stage_map;
    uint32_t off = 0;
    g.blob = off;
    off = align_up(off + g.B.bytes, 16);
    g.map = off;
    if (stage_map) off = align_up(off + (uint32_t)(lsb * (lsb + 1) / 2 + 8) * 2u, 16);
    g.sp = off;
    off = align_up(off + (uint32_t)(sd + 1) * 8u, 16);
    g.acc = off;
    off = align_up(off + (uint32_t)(lsb * (lsb + 1) / 2) * 8u, 16);
    g.rhs = off;
    off += (uint32_t)lsb * 8u;
    g.hits = off;
    off = align_up(off + (uint32_t)lsb * 4u, 16);
    g.gath = off;  // gx, gy, gz [CNB * 8] doubles, gi [CNB * 8] u16
    off = align_up(off + (uint32_t)CNB * 8u * 26u, 16);
    g.phi = off;   // [CKS][CNB][32] doubles
    off += (uint32_t)CKS * CNB * 32u * 8u;
    g.misc = off;  // claimed items
    off += 16;
    g.region = align_up(off, 128);
    return g;
}

// Static split of the NB(NB+1)/2 upper blocks (row-major) into CW ranges.
__host__ __device__ constexpr int cta_nblk(int nb) { return nb * (nb + 1) / 2; }
__host__ __device__ constexpr int cta_bw(int nb) { return (cta_nblk(nb) + CW - 1) / CW; }
__host__ __device__ constexpr int cta_tri_I(int n, int idx) {
    int I = 0;
    while (idx >= n - I) {
        idx -= n - I;
        ++I;
    }
    return I;
}
__host__ __device__ constexpr int cta_tri_J(int n, int idx) {
    int I = 0;
    while (idx >= n - I) {
        idx -= n - I;
        ++I;
    }
    return I + idx;
}

template <int N, typename F, int... Is>
__device__ __forceinline__ void cta_static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void cta_static_for(F&& f) {
    cta_static_for_impl<N>(f, std::make_integer_sequence<int, N>{});
}

struct CtaSub {
    const double* gx;
    const double* gy;
    const double* gz;
    const uint16_t* gi;
    int Ls;
    uint64_t q0, q1;
};

// SYRK of warp W over one chunk of ks k-steps: blocks [W*BW, min(T, (W+1)*BW)).
template <int NB, int W>
__device__ __forceinline__ void cta_syrk(const double* phi, int ks, int lane, double (&acc)[cta_bw(CNB)][2]) {
    constexpr int T = cta_nblk(NB), BW = cta_bw(NB), B0 = W * BW;
    constexpr int NBLK = (B0 + BW <= T) ? BW : (T > B0 ? T - B0 : 0);
    if constexpr (NBLK > 0) {
        for (int s = 0; s < ks; ++s) {
            double f[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) f[i] = phi[(s * NB + i) * 32 + lane];
            cta_static_for<NBLK>([&](auto tc) {
                constexpr int t = decltype(tc)::value;
                constexpr int I = cta_tri_I(NB, B0 + t), J = cta_tri_J(NB, B0 + t);
                dmma_8x8x4(acc[t], f[I], f[J]);
            });
        }
    }
}

// Fold of warp W's register blocks into the shared accumulator.
template <int NB, int W>
__device__ __forceinline__ void cta_fold(const CtaSub& S, double* A, uint32_t LS, int lane,
                                         const double (&acc)[cta_bw(CNB)][2]) {
    constexpr int T = cta_nblk(NB), BW = cta_bw(NB), B0 = W * BW;
    constexpr int NBLK = (B0 + BW <= T) ? BW : (T > B0 ? T - B0 : 0);
    if constexpr (NBLK > 0) {
        const int rs = lane >> 2, kq = lane & 3;
        uint32_t ad[2 * NBLK];
        bool ok[2 * NBLK];
        double old[2 * NBLK];
        cta_static_for<NBLK>([&](auto tc) {
            constexpr int t = decltype(tc)::value;
            constexpr int I = cta_tri_I(NB, B0 + t), J = cta_tri_J(NB, B0 + t);
            const int a = I * 8 + rs;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = J * 8 + 2 * kq + e;
                ok[2 * t + e] = a < S.Ls && c < S.Ls && (J > I || rs <= 2 * kq + e);
                ad[2 * t + e] = ok[2 * t + e] ? row_off(S.gi[a], LS) + S.gi[c] : 0u;
            }
        });
#pragma unroll
        for (int k = 0; k < 2 * NBLK; ++k) old[k] = ok[k] ? A[ad[k]] : 0.0;
#pragma unroll
        for (int k = 0; k < 2 * NBLK; ++k)
            if (ok[k]) A[ad[k]] = old[k] + acc[k / 2][k % 2];
    }
}

// One sub-tile with NB blocks: phi chunks, SYRK, fold, A^T h / hits.
template <int DIM, int FAM, int NB>
__device__ __forceinline__ void cta_subtile(const AsmParams& P, const CtaSub& S, double* phi, double* A, double* R,
                                            uint32_t* H, uint32_t LS, int warp, int lane) {
    constexpr int NO = (NB + CW - 1) / CW;  // phi blocks owned per warp (I = warp + CW o)
    const int rs = lane >> 2, kq = lane & 3;
    double acc[cta_bw(CNB)][2];
#pragma unroll
    for (int t = 0; t < cta_bw(CNB); ++t) acc[t][0] = acc[t][1] = 0.0;
    double rh[NO];
    uint32_t hc[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        rh[o] = 0.0;
        hc[o] = 0u;
    }
    for (uint64_t c0 = S.q0; c0 < S.q1; c0 += 4 * CKS) {
        const uint64_t rem_steps = (S.q1 - c0 + 3) / 4;
        const int ks = rem_steps < (uint64_t)CKS ? (int)rem_steps : CKS;
        // ---- phi phase: fragments (s, I) of this warp's row blocks
        for (int s = 0; s < ks; ++s) {
            const double4 p = point_rec(P, c0 + 4 * s + kq, S.q1, DIM);
            const double h = DIM == 2 ? p.z : p.w;
#pragma unroll
            for (int o = 0; o < NO; ++o) {
                const int I = warp + CW * o;
                if (I < NB) {
                    const int a = I * 8 + rs;
                    bool in;
                    const double f = phi_at<DIM, FAM>(p.x, p.y, p.z, S.gx[a], S.gy[a], DIM == 3 ? S.gz[a] : 0.0,
                                                      P.alpha, P.incl_bits, in);
                    phi[(s * NB + I) * 32 + lane] = f;
                    rh[o] = fma(f, h, rh[o]);
                    hc[o] += in ? 1u : 0u;
                }
            }
        }
        __syncthreads();
        // ---- SYRK phase
        switch (warp) {
            case 0: cta_syrk<NB, 0>(phi, ks, lane, acc); break;
            case 1: cta_syrk<NB, 1>(phi, ks, lane, acc); break;
            case 2: cta_syrk<NB, 2>(phi, ks, lane, acc); break;
            default: cta_syrk<NB, 3>(phi, ks, lane, acc);
        }
        if (c0 + 4 * CKS < S.q1) __syncthreads();  // the fragment buffer is refilled
    }
    // ---- fold (disjoint blocks per warp) and the rows' A^T h / hits (disjoint rows)
    switch (warp) {
        case 0: cta_fold<NB, 0>(S, A, LS, lane, acc); break;
        case 1: cta_fold<NB, 1>(S, A, LS, lane, acc); break;
        case 2: cta_fold<NB, 2>(S, A, LS, lane, acc); break;
        default: cta_fold<NB, 3>(S, A, LS, lane, acc);
    }
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        rh[o] += __shfl_xor_sync(0xffffffffu, rh[o], 1);
        hc[o] += __shfl_xor_sync(0xffffffffu, hc[o], 1);
        rh[o] += __shfl_xor_sync(0xffffffffu, rh[o], 2);
        hc[o] += __shfl_xor_sync(0xffffffffu, hc[o], 2);
        const int a = (warp + CW * o) * 8 + rs;
        if (warp + CW * o < NB && kq == 0 && a < S.Ls && hc[o]) {
            const uint16_t g = S.gi[a];
            R[g] += rh[o];
            H[g] += hc[o];
        }
    }
}

template <int DIM, int FAM>
__global__ void __launch_bounds__(CT, 4)
    assemble_cta_kernel(AsmParams P, CGeom G, const uint32_t* __restrict__ items,
                        const unsigned char* __restrict__ blobs, uint32_t n_items, unsigned* __restrict__ work) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int SD = P.SD;
    double* A = reinterpret_cast<double*>(sm + G.acc);
    double* R = reinterpret_cast<double*>(sm + G.rhs);
    uint32_t* H = reinterpret_cast<uint32_t*>(sm + G.hits);
    double* gx = reinterpret_cast<double*>(sm + G.gath);
    double* gy = gx + CNB * 8;
    double* gz = gy + CNB * 8;
    uint16_t* gi = reinterpret_cast<uint16_t*>(gz + CNB * 8);
    double* phi = reinterpret_cast<double*>(sm + G.phi);
    uint32_t* claim = reinterpret_cast<uint32_t*>(sm + G.misc);
    const unsigned char* Bl = sm + G.blob;
    const uint32_t* subt = reinterpret_cast<const uint32_t*>(Bl + G.B.sub);
    const double* cx = reinterpret_cast<const double*>(Bl + G.B.cx);
    const double* cy = reinterpret_cast<const double*>(Bl + G.B.cy);
    const double* cz = reinterpret_cast<const double*>(Bl + G.B.cz);
    const uint16_t* lists = reinterpret_cast<const uint16_t*>(Bl + G.B.lists);
    const uint64_t* up = reinterpret_cast<const uint64_t*>(Bl + G.B.uptr);
    const uint32_t* cid = reinterpret_cast<const uint32_t*>(Bl + G.B.cid);
    uint64_t* sp = reinterpret_cast<uint64_t*>(sm + G.sp);
    uint16_t* map_s = reinterpret_cast<uint16_t*>(sm + G.map);

    if (tid == 0) claim[0] = atomicAdd(work, 1u);
    __syncthreads();
    uint32_t it = claim[0];
    while (it < n_items) {
        const uint32_t T = items[it];
        const uint64_t key0 = (uint64_t)T * (uint64_t)SD;
        __syncthreads();  // everyone has read claim[0] / finished the previous super-tile
        if (tid == 0) claim[0] = atomicAdd(work, 1u);
        // ---- stage the blob and the sub-tile ranges; the slot map follows asynchronously
        for (int i = tid; i <= SD; i += CT) sp[i] = P.pptr[key0 + i];
        {
            const int4* src = reinterpret_cast<const int4*>(blobs + (size_t)it * G.B.bytes);
            int4* dst = reinterpret_cast<int4*>(sm + G.blob);
            for (uint32_t i = tid; i < G.B.bytes / 16u; i += CT) dst[i] = __ldg(src + i);
        }
        __syncthreads();
        const uint32_t nit = claim[0];
        if (nit < n_items && warp == CW - 1) {  // pull the next blob towards L2
            const unsigned char* nb = blobs + (size_t)nit * G.B.bytes;
            for (uint32_t o = lane * 128u; o < G.B.bytes; o += 32u * 128u)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(nb + o));
        }
        if (sp[0] == sp[SD]) {  // no points in this super-tile
            it = nit;
            continue;
        }
        const uint32_t LS = *reinterpret_cast<const uint32_t*>(Bl);
        const uint16_t* gmap = P.smap + P.smptr[T];
        if (G.map_staged) {
            const uint32_t n16 = (LS * (LS + 1) / 2 + 7) / 8;
            for (uint32_t i = tid; i < n16; i += CT)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(map_s + 8 * i)),
                             "l"(gmap + 8 * i)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        {
            const uint32_t nacc = LS * (LS + 1) / 2;
            for (uint32_t i = tid; i < nacc; i += CT) A[i] = 0.0;
            for (uint32_t i = tid; i < LS; i += CT) {
                R[i] = 0.0;
                H[i] = 0u;
            }
        }
        // ---- sub-tiles
        for (int j = 0; j < SD; ++j) {
            CtaSub S;
            S.q0 = sp[j];
            S.q1 = sp[j + 1];
            const uint32_t st = subt[j];
            S.Ls = (int)(st >> 16);
            if (S.q0 == S.q1 || S.Ls == 0) continue;  // uniform across the CTA
            const uint16_t* list = lists + (st & 0xffffu);
            const int NB = (S.Ls + 7) >> 3;
            __syncthreads();  // previous sub-tile done with the gather arrays (and the accumulator zeroed)
            for (int a = tid; a < NB * 8; a += CT) {
                if (a < S.Ls) {
                    const int Aidx = list[a];
                    gx[a] = cx[Aidx];
                    gy[a] = cy[Aidx];
                    if (DIM == 3) gz[a] = cz[Aidx];
                    gi[a] = (uint16_t)Aidx;
                } else {
                    gx[a] = kFar;
                    gy[a] = kFar;
                    if (DIM == 3) gz[a] = kFar;
                    gi[a] = 0;
                }
            }
            __syncthreads();
            S.gx = gx;
            S.gy = gy;
            S.gz = gz;
            S.gi = gi;
            switch (NB) {
                case 1: cta_subtile<DIM, FAM, 1>(P, S, phi, A, R, H, LS, warp, lane); break;
                case 2: cta_subtile<DIM, FAM, 2>(P, S, phi, A, R, H, LS, warp, lane); break;
                case 3: cta_subtile<DIM, FAM, 3>(P, S, phi, A, R, H, LS, warp, lane); break;
                case 4: cta_subtile<DIM, FAM, 4>(P, S, phi, A, R, H, LS, warp, lane); break;
                case 5: cta_subtile<DIM, FAM, 5>(P, S, phi, A, R, H, LS, warp, lane); break;
                case 6: cta_subtile<DIM, FAM, 6>(P, S, phi, A, R, H, LS, warp, lane); break;
                case 7: cta_subtile<DIM, FAM, 7>(P, S, phi, A, R, H, LS, warp, lane); break;
                default: cta_subtile<DIM, FAM, 8>(P, S, phi, A, R, H, LS, warp, lane);
            }
        }
        if (G.map_staged) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        // ---- flush: one global fp64 reduction per nonzero pair of the super-tile
        {
            const uint16_t* map = G.map_staged ? map_s : gmap;
            const uint32_t nacc = LS * (LS + 1) / 2;
            uint32_t Ar = 0, rend = LS;  // row of entry e and the end of that row
            constexpr int FB = 4;
            for (uint32_t e0 = tid; e0 < nacc; e0 += CT * FB) {
                uint16_t off[FB];
                double v[FB];
#pragma unroll
                for (int k = 0; k < FB; ++k) {
                    const uint32_t e = e0 + CT * k;
                    off[k] = e < nacc ? (G.map_staged ? map[e] : __ldg(map + e)) : (uint16_t)0;
                    v[k] = e < nacc ? A[e] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < FB; ++k) {
                    const uint32_t e = e0 + CT * k;
                    if (e >= nacc) break;
                    while (e >= rend) {
                        ++Ar;
                        rend += LS - Ar;
                    }
                    if (v[k] != 0.0) {
                        if (off[k] == 0xffffu) atomicAdd(P.miss, 1ull);
                        else red_add(P.vals + up[Ar] + off[k], v[k]);
                    }
                }
            }
        }
        for (uint32_t a = tid; a < LS; a += CT) {
            const uint32_t hc = H[a];
            if (hc) {
                red_add(P.rhs + cid[a], R[a]);
                red_add(P.hits + cid[a], (double)hc);
            }
        }
        it = nit;
    }
}

}  // namespace
}  // namespace rbg
