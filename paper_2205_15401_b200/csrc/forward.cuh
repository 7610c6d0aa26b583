// K3: fused per-pixel trace -> eta filter -> K'-nearest selection -> closed-form blend.
#pragma once

#include "gvr_common.cuh"

namespace gvrk {

// FP32 constants of the q classification (classify_key), set on the host.
struct QClass {
    float c_rej, c_acc;   // 2(-ln eta + g), 2(-ln eta - g)
    float slack_lo, slack_hi;  // 1 -/+ relative slack
    float f, inv_f;       // F, 1 / F
};

struct FwdParams {
    CameraP cam;
    SelP sel;
    int D, Dc;
    double tau;
    float guard_abs;     // FP32 guard band on q (absolute)
    float prefilter_c1;  // 1 - relative slack on delta.S.delta
    QClass qc;           // classification constants (from guard_abs, prefilter_c1, ln eta, F)
    int exact_only;      // test hook: every candidate through the exact FP64 trace
    int tiles_x;
    const int* tile_order;  // tiles by list length, longest first (LPT); first *n_order valid
    const int* n_order;
    const int* tile_count;           // [tiles] list lengths
    const int* tile_off;             // [tiles] list offset in the pool; -1: not listed (pool overflow:
                                     // the tile streams every kernel through the same exact tests)
    const unsigned long long* pool;  // tile lists (order(zmin) << 32 | id), unsorted within a list
    unsigned long long* sorted_pool; // same offsets: sorted copies of lists too long for shared memory
    int list_smem;                   // lists up to this length are sorted in shared memory (<= kSelListSmem)
    int K;
    const int* tile_order_blend;  // tiles by sum_p n_p^2 (from the selection), then the tiles with no
    const int* n_order_blend;     // selection (cleared by the blend); first *n_order_blend valid
    const Rec32* rec32;
    const Rec64* rec64;
    const double* attr;  // [K*D] object attributes (FP64)
    // outputs
    double* image;  // [P*Dc]
    double* alpha;  // [P]
    double* depth;  // [P]
    int* topk;      // [P*kp], first count[p] valid
    int* count;     // [P]
    double* topk_w; // [P*kp] or null
    double* tape_t; // [P*kp] T(l_k) of the selected entries (backward input)
    EntryRec* ent;  // [P*kp] traced selected entries (written by the blend)
    double* ent_a;  // [P*kp] a = d.Sd of each selected entry (FP64, the backward's chain)
    int presorted;   // topk already in exact (l, idx) order (warp selection); else the blend sorts
    unsigned* tile_done;     // [tiles] set (release) when the tile's selection is written; the blend,
                             // launched as a programmatic dependent, waits per tile (nullable)
    long long* tile_cycles;  // profiling hook: [tiles] SM cycles of the tile's selection CTA (nullable)
    unsigned* tile_hint;     // [tiles] out: the same cycles, the LPT costs of the next render of this view
    int precise;     // verification mode: FP64 exact traces and erfc in the blend sums (gradcheck)
    int* nonfinite; // flag
    const int4* kinfo;          // [K] mask rectangles (project_kernel)
    unsigned long long* masks;  // (kernel, tile) pixel masks for the backward
};

// FP32 centre-relative classification of q against ln(eta), and the FP32
// depth key of the certain accepts.
// With dt = ((i-Oy)/F, (j-Ox)/F, 1), delta = m - z dt = (z/F)(c_i - i, c_j - j, 0)
// is formed without cancellation from the integer and fractional parts of the
// projected centre, and (the line minimum is parametrisation independent)
//   q = -T / (2A),  T = delta.S.delta * A - (dt.S.delta)^2 >= 0,  A = dt.S.dt > 0.
// Division-free, with a guard band g on q and a relative slack on the
// delta.S.delta * A term (FP32 cancellation):
//   returns 0: q <= ln(eta) for certain      (reject)
//           2: q >  ln(eta) for certain      (eligible; *key set)
//           1: inside the band, or a key     (decide with the exact FP64 trace)
//              whose error bound is not met
// Depth key: the minimiser along dt is t* = z + B'/A (m = z dt + delta, B' =
// dt.S.delta), so l = |dt| t* = nrm (z + (z/F) c), c = (di sd0 + dj sd1) / A
// with (di, dj) = (c_i - i, c_j - j) in pixels. In FP32 the key is within
// 6 units of 2^-24 |l| of the exact l (z: 1, c: <= 2 by the checked bound
// below, fma + product: 2, nrm: 1), so keys more than kKeyClose apart order
// like the exact keys and closer ones are decided on the exact trace.

__device__ __forceinline__ int classify_key(const Rec32& r, int i, int j, float u, float v, float nrm,
                                            const QClass& qc, float* key) {
    if (r.z < 0.0f) return 1;  // unusual geometry: exact path only
    const float zf = r.z * qc.inv_f;
    const float di = (float)(r.ci_int - i) + r.ci_frac;
    const float dj = (float)(r.cj_int - j) + r.cj_frac;
    const float dx = zf * di, dy = zf * dj;
    const float sd0 = fmaf(r.s00, u, fmaf(r.s01, v, r.s02));
    const float sd1 = fmaf(r.s01, u, fmaf(r.s11, v, r.s12));
    const float sd2 = fmaf(r.s02, u, fmaf(r.s12, v, r.s22));
    const float A = fmaf(u, sd0, fmaf(v, sd1, sd2));
    const float Bp = fmaf(di, sd0, dj * sd1);
    const float B = zf * Bp;
    const float dsd = fmaf(dx, fmaf(r.s00, dx, 2.0f * r.s01 * dy), r.s11 * dy * dy);
    const float bb = B * B;
    if (fmaf(dsd * qc.slack_lo, A, -bb) > qc.c_rej * A) return 0;
    if (!(fmaf(dsd * qc.slack_hi, A, -bb) < qc.c_acc * A)) return 1;
    if (key) {
        const float rA = 1.0f / A;
        const float c = Bp * rA;
        // error of c (each FP32 rounding of S, (u, v), (di, dj), the sums and the
        // quotient; 8 units of 2^-24 of the unsigned sums) must stay within 2
        // units of 2^-24 of F + c >= F / 2: (Babs + |c| Aabs) / A <= F / 8
        const float a0 = fabsf(r.s00 * u) + fabsf(r.s01 * v) + fabsf(r.s02);
        const float a1 = fabsf(r.s01 * u) + fabsf(r.s11 * v) + fabsf(r.s12);
        const float a2 = fabsf(r.s02 * u) + fabsf(r.s12 * v) + fabsf(r.s22);
        const float babs = (fabsf(di) + 1.0f) * a0 + (fabsf(dj) + 1.0f) * a1;
        const float aabs = fabsf(u) * a0 + fabsf(v) * a1 + a2;
        if (!(fmaf(fabsf(c), aabs, babs) * rA <= 0.125f * qc.f) || !(fabsf(c) <= 0.5f * qc.f)) return 1;
        *key = nrm * fmaf(zf, c, r.z);
    }
    return 2;
}

__device__ __forceinline__ int classify_q(const Rec32& r, int i, int j, float u, float v, const QClass& qc) {
    return classify_key(r, i, j, u, v, 1.0f, qc, nullptr);
}

// Loads a tile's candidate list into shared memory in ascending order of a
// depth bound: a CTA counting sort over 256 buckets spanning the tile's own
// zmin range (3 passes over the list, 4 barriers; entries inside a bucket stay
// in arbitrary order). The high word of each key is replaced by its bucket's
// lower bound, so keys[e] >> 32 is non-decreasing along the list and bounds the
// zmin (hence the l) of every entry at or after e -- all the early exit needs.
// The selection itself is exact and independent of the visiting order.
// Returns the list length, or -1 when the tile's list did not fit the pool (the
// caller then streams every kernel, unsorted, with the same exact tests).
// Lists longer than smem_cap are sorted into the tile's slot of the global
// sorted pool instead of shared memory; *list points at the sorted list.
// With `stage` (>= smem_cap + 2 entries of shared memory), a list that fits is
// first brought into shared memory with one TMA bulk copy (cp.async.bulk,
// completing on an mbarrier), and the three sort passes read it there.
__device__ __forceinline__ int load_sorted_list(const FwdParams& p, int tile, unsigned long long* keys,
                                                int smem_cap, const unsigned long long** list,
                                                unsigned long long* stage = nullptr) {
    constexpr int NB = 256;
    __shared__ unsigned s_lo, s_hi;
    __shared__ int s_hist[NB];
    const int count = p.tile_count[tile];
    const int off = p.tile_off[tile];
    if (off < 0) return count > 0 ? -1 : 0;
    const unsigned long long* src = p.pool + off;
    if (count > smem_cap) keys = p.sorted_pool + off;
    *list = keys;
    __shared__ __align__(8) unsigned long long s_mbar;
    const bool bulk = stage && count > 0 && count <= smem_cap;
    const int a0 = off & ~1;  // 16-byte aligned source (the pool keeps 2 entries of slack at its end)
    if (threadIdx.x == 0) {
        s_lo = 0xffffffffu;
        s_hi = 0u;
        if (bulk) {
            const unsigned bytes = (unsigned)(((off + count - a0) * 8 + 15) & ~15);
            mbar_init(&s_mbar, 1);
            mbar_expect_tx(&s_mbar, bytes);
            bulk_copy_g2s(stage, p.pool + a0, bytes, &s_mbar);
        }
    }
    for (int b = threadIdx.x; b < NB; b += blockDim.x) s_hist[b] = 0;
    __syncthreads();
    if (bulk) {
        mbar_wait(&s_mbar, 0);
        src = stage + (off - a0);
    }
    unsigned lo = 0xffffffffu, hi = 0u;
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        const unsigned z = (unsigned)(src[e] >> 32);
        lo = min(lo, z);
        hi = max(hi, z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0 && count > 0) {
        atomicMin(&s_lo, lo);
        atomicMax(&s_hi, hi);
    }
    __syncthreads();
    lo = s_lo;
    const unsigned range = count > 0 ? s_hi - lo : 0u;
    int shift = 0;
    while ((range >> shift) >= (unsigned)NB) ++shift;
    for (int e = threadIdx.x; e < count; e += blockDim.x)
        atomicAdd(&s_hist[((unsigned)(src[e] >> 32) - lo) >> shift], 1);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 buckets, 8 per lane
        int vals[8], run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            vals[q] = s_hist[threadIdx.x * 8 + q];
            run += vals[q];
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (threadIdx.x >= o) incl += y;
        }
        int base = incl - run;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            s_hist[threadIdx.x * 8 + q] = base;
            base += vals[q];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        const unsigned long long k = src[e];
        const unsigned b = ((unsigned)(k >> 32) - lo) >> shift;
        const unsigned long long bound = (unsigned long long)(lo + (b << shift));
        keys[atomicAdd(&s_hist[b], 1)] = (bound << 32) | (k & 0xffffffffull);
    }
    __syncthreads();
    return count;
}

#ifndef GVR_SEL_LIST_SMEM
#define GVR_SEL_LIST_SMEM 2048
#endif
constexpr int kSelListSmem = GVR_SEL_LIST_SMEM;  // sorted tile list entries kept in shared memory

// Per-warp candidate chunk entry.
struct __align__(16) Cand {
    Rec32 r;
    int k;
    int pad[3];
};

// Fast FP64 peak distance l = b / a with the reference's a = d.Sd and
// b = (m.Sd + d.Sm) / 2 (full S), contracted FMAs: within a few ulps (~1e-15
// relative) of the reference-order l of trace_exact. Keys of the CTA selection
// (K' > 32).
__device__ __forceinline__ double fast_l(const Rec64& r, const double* d) {
    const double* s = r.s;
    const double sd0 = fma(s[0], d[0], fma(s[1], d[1], s[2] * d[2]));
    const double sd1 = fma(s[3], d[0], fma(s[4], d[1], s[5] * d[2]));
    const double sd2 = fma(s[6], d[0], fma(s[7], d[1], s[8] * d[2]));
    const double a = fma(d[0], sd0, fma(d[1], sd1, d[2] * sd2));
    const double b = 0.5 * (fma(r.m[0], sd0, fma(r.m[1], sd1, r.m[2] * sd2)) +
                            fma(d[0], r.sm[0], fma(d[1], r.sm[1], d[2] * r.sm[2])));
    double rc;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(a));
    rc = rc * fma(-a, rc, 2.0);  // Newton: ~2^-40
    rc = rc * fma(-a, rc, 2.0);  // ~1 ulp
    return b * rc;
}

// Selection keys: (l, id) where l is either the fast l (error < 1e-11 |l|, a
// 10^4 safety factor over the few-ulp actual error) or the exact reference l
// (id carries kExact). Two keys closer than the error bound are upgraded to
// exact before comparing, so every decision equals the reference's (l, idx) order.
constexpr int kExact = 0x40000000;

__device__ __forceinline__ bool keys_close(double a, double b) { return fabs(a - b) <= 1e-11 * fabs(a) + 1e-300; }

__device__ __forceinline__ void make_exact(double& l, int& id, const double* d, const Rec64* rec64) {
    if (!(id & kExact)) {
        l = trace_exact(d, rec64[id]).l;
        id |= kExact;
    }
}

// (la, ia) < (lb, ib) in the reference order; may upgrade either key to exact.
__device__ __forceinline__ bool key_less(double& la, int& ia, double& lb, int& ib, const double* d,
                                         const Rec64* rec64) {
    if (!keys_close(la, lb)) return la < lb;
    make_exact(la, ia, d, rec64);
    make_exact(lb, ib, d, rec64);
    return la < lb || (la == lb && (ia & ~kExact) < (ib & ~kExact));
}

// Worst (largest key) of the n kept entries of this thread; upgrades near ties in place.
__device__ __forceinline__ void find_worst(double* s_l, int* s_id, int n, int tid, const double* d,
                                           const Rec64* rec64, double& wl, int& wid, int& wslot) {
    wl = s_l[tid];
    wid = s_id[tid];
    wslot = 0;
    for (int s = 1; s < n; ++s) {
        double ls = s_l[s * 64 + tid];
        int is = s_id[s * 64 + tid];
        const int was_w = wid, was_s = is;
        const bool less = key_less(wl, wid, ls, is, d, rec64);
        if (wid != was_w) {  // upgraded: write back
            s_l[wslot * 64 + tid] = wl;
            s_id[wslot * 64 + tid] = wid;
        }
        if (is != was_s) {
            s_l[s * 64 + tid] = ls;
            s_id[s * 64 + tid] = is;
        }
        if (less) {
            wl = ls;
            wid = is;
            wslot = s;
        }
    }
}

// K3a selection. CTA = one 8x8 pixel tile = 2 warps that stream the tile's
// list independently (no CTA barriers; a warp stops as soon as its 32 pixels
// are done). Per candidate: exact box test (pixel centre inside the eta box),
// FP32 classification of q (exact FP64 trace only inside the guard band), then
// the K' nearest by key (fast l, exact on near ties) are kept UNSORTED in shared
// memory with the current worst tracked in registers. The blend kernel sorts
// the set by exact (l, idx).
template <int KMAX>
__global__ void __launch_bounds__(64) select_kernel(FwdParams p) {
    constexpr int TILE = 8, NT = 64;
    extern __shared__ __align__(16) unsigned char smem[];
    Cand* chunk = reinterpret_cast<Cand*>(smem) + (threadIdx.x & ~31);
    double* s_l = reinterpret_cast<double*>(smem + sizeof(Cand) * NT);
    int* s_id = reinterpret_cast<int*>(s_l + KMAX * NT);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(s_id + KMAX * NT);

    if ((int)blockIdx.x >= *p.n_order) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const int tile = p.tile_order[blockIdx.x];
    const int i = (tile / p.tiles_x) * TILE + tid / TILE;
    const int j = (tile % p.tiles_x) * TILE + tid % TILE;
    const bool inside = i < p.cam.H && j < p.cam.W;
    const unsigned long long* tl = keys;
    const int listed = load_sorted_list(p, tile, keys, p.list_smem, &tl);
    const bool overflow = listed < 0;  // stream every kernel, unsorted
    const int start = 0;
    const int end = overflow ? p.K : listed;
    const long long pix = (long long)i * p.cam.W + j;
    const int kp = p.sel.kp;

    double d[3];
    pixel_ray(p.cam, inside ? i : 0, inside ? j : 0, d);
    const float u = (float)xdiv(xsub((double)i, p.cam.oy), p.cam.focal);
    const float v = (float)xdiv(xsub((double)j, p.cam.ox), p.cam.focal);
    const float fi = (float)i, fj = (float)j;
    const QClass& qc = p.qc;  // kernel parameter space: no registers
    const bool exact_only = p.exact_only != 0;
    const double log_eta = p.sel.log_eta;
    const Rec64* rec64 = p.rec64;

    // selection state: n kept; once full, the worst kept key and its slot
    int n = 0, wslot = 0, wid = 0x7fffffff;
    double wl = INFINITY;
    bool done = !inside;

    for (int base = start; base < end; base += 32) {
        if (__all_sync(0xffffffffu, done)) break;
        const int e = base + lane;
        if (e < end) {
            const int k = overflow ? e : (int)(tl[e] & 0xffffffffu);
            chunk[lane].r = p.rec32[k];
            chunk[lane].k = k;
        }
        __syncwarp();
        const int cnt = min(32, end - base);
        for (int c0 = 0; c0 < cnt && !done; c0 += 4) {
            // early exit: every later candidate has l >= zmin > worst kept (+ key error)
            if (!overflow &&
                (double)float_from_order_bits((uint32_t)(tl[base + c0] >> 32)) > wl + 1e-11 * fabs(wl)) {
                done = true;
                break;
            }
            int cls[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const Rec32& r = chunk[min(c0 + q, cnt - 1)].r;
                const bool in_box = c0 + q < cnt && fi >= r.top && fi <= r.bottom && fj >= r.left && fj <= r.right;
                cls[q] = in_box ? classify_q(r, i, j, u, v, qc) : 0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (cls[q] == 0) continue;
                int k = chunk[c0 + q].k;
                double lk;
                if (exact_only || cls[q] == 1) {
                    const Traced64 t = trace_exact(d, rec64[k]);
                    if (!(t.q > log_eta)) continue;  // fine_select threshold (tracer.cpp:117-118)
                    lk = t.l;
                    k |= kExact;
                } else {
                    lk = fast_l(rec64[k], d);
                }
                if (n < kp) {
                    s_l[n * NT + tid] = lk;
                    s_id[n * NT + tid] = k;
                    if (++n == kp) find_worst(s_l, s_id, n, tid, d, rec64, wl, wid, wslot);
                } else {
                    const int was_w = wid;
                    const bool better = key_less(lk, k, wl, wid, d, rec64);
                    if (better) {
                        s_l[wslot * NT + tid] = lk;
                        s_id[wslot * NT + tid] = k;
                        find_worst(s_l, s_id, n, tid, d, rec64, wl, wid, wslot);
                    } else if (wid != was_w) {  // the worst was upgraded to exact
                        s_l[wslot * NT + tid] = wl;
                        s_id[wslot * NT + tid] = wid;
                    }
                }
            }
        }
        __syncwarp();
    }

    if (!inside) return;
    for (int s = 0; s < n; ++s) p.topk[pix * kp + s] = s_id[s * NT + tid] & ~kExact;  // unsorted; the blend sorts
    p.count[pix] = n;
}

#ifndef GVR_SEL_WARP_LIST
#define GVR_SEL_WARP_LIST 512
#endif
constexpr int kWarpListCap = GVR_SEL_WARP_LIST;  // per-warp compacted list capacity (entries)

// Exact order of two selection candidates (kernel ids a, b; l on the exact trace).
__device__ __forceinline__ bool exact_less(int a, int b, const double* d, const Rec64* rec64) {
    const double la = trace_exact(d, rec64[a]).l, lb = trace_exact(d, rec64[b]).l;
    return la < lb || (la == lb && a < b);
}

// FP32 rank keys (classify_key, or the exact l rounded to FP32): within 7 units
// of 2^-24 |l| of the exact l, so two keys farther apart than kKeyClose |l|
// order like the exact keys; closer ones are compared on the exact trace.
constexpr float kKeyClose = 9.5367431640625e-7f;  // 2^-20 = 16 units of 2^-24

__device__ __forceinline__ bool keyf_close(float a, float b) { return fabsf(a - b) <= kKeyClose * fabsf(b); }

#ifndef GVR_SEL_CUNROLL  // list batches per compaction step (loads in flight together)
#define GVR_SEL_CUNROLL 4
#endif
#ifndef GVR_SEL_BATCH_MIN  // eligible candidates per batch from which the batch merge is used (33: never)
#define GVR_SEL_BATCH_MIN 10
#endif
// Keys within kKeyUlps units in the last place of each other are "close" for the
// batch merge: 16 ulps >= 16 * 2^-24 |l| > the sum of two keys' errors (<= 14
// units), so keys farther apart order like the exact keys.
constexpr unsigned kKeyUlps = 16u;

// Batch merge of one 32-candidate batch into the kept list (warp-wide): bitonic
// sort of the eligible candidates by (FP32 key, id), binary-search ranks of
// candidates among the kept entries and of kept entries among the candidates,
// scatter into sl/si (candidates flagged in bit 31 of the id). The merge is
// exact unless an entry adjacent to a candidate in the merged order (up to the
// first dropped position) lies within kKeyUlps of it: then it returns false and
// the caller ranks the batch one candidate at a time on the exact trace.
// Replaces ~35 warp instructions per eligible candidate with ~160 per batch.
// Ascending bitonic sort of one 64-bit key per lane within groups of W lanes.
template <int W>
__device__ __forceinline__ unsigned long long bitonic_lanes(unsigned long long ck, int lane) {
#pragma unroll
    for (int size = 2; size <= W; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, ck, stride);
            const bool asc = size == W || (lane & size) == 0;
            const bool lower = (lane & stride) == 0;
            ck = (lower == asc) ? (o < ck ? o : ck) : (o > ck ? o : ck);
        }
    }
    return ck;
}

__device__ __forceinline__ bool merge_batch(float L, int I, int n, float lk, int k, bool me, int m, int kp, int lane,
                                            float* sl, int* si) {
    const unsigned FULL = 0xffffffffu;
    unsigned long long ck = me ? ((unsigned long long)float_order_bits(lk) << 32) | (unsigned)k : ~0ull;
    if (m <= 16) {
        // compact the eligible candidates to lanes 0..m-1 (staged in the upper
        // half of the warp's list): a 16-lane sort (10 stages instead of 15)
        const int r = __popc(__ballot_sync(FULL, me) & ((1u << lane) - 1u));
        if (me) {
            sl[32 + r] = lk;
            si[32 + r] = k;
        }
        __syncwarp();
        ck = lane < m ? ((unsigned long long)float_order_bits(sl[32 + lane]) << 32) | (unsigned)si[32 + lane] : ~0ull;
        __syncwarp();
        ck = bitonic_lanes<16>(ck, lane);
    } else {
        ck = bitonic_lanes<32>(ck, lane);
    }
    const unsigned cu = (unsigned)(ck >> 32);  // lane r < m: key of the r-th smallest candidate
    if (n == 0) {
        // nothing kept yet (a pixel's first eligible batch): the sorted
        // candidates are the merged order; only their adjacency is checked
        const unsigned nxt = __shfl_down_sync(FULL, cu, 1);
        const bool bad = lane + 1 < min(m, kp + 1) && nxt - cu <= kKeyUlps;
        if (__any_sync(FULL, bad)) return false;
        if (lane < min(m, kp)) {
            sl[lane] = float_from_order_bits(cu);
            si[lane] = (int)(unsigned)ck;
        }
        __syncwarp();
        return true;
    }
    const unsigned ku = float_order_bits(L);   // lane s < n: key of kept entry s (non-decreasing)
    // below: kept entries at or before the candidate (ties: kept first); above: candidates before the kept entry
    int below = 0, above = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1) {
        const int pb = below + step, pa = above + step;
        const unsigned kv = __shfl_sync(FULL, ku, (pb - 1) & 31);
        const unsigned cv = __shfl_sync(FULL, cu, (pa - 1) & 31);
        if (pb <= n && kv <= cu) below = pb;
        if (pa <= m && cv < ku) above = pa;
    }
    const int lim = min(n + m, kp + 1);  // merged positions kept, plus the first dropped one
    if (lane < m && lane + below < lim) {
        sl[lane + below] = float_from_order_bits(cu);
        si[lane + below] = (int)((unsigned)ck | 0x80000000u);
    }
    if (lane < n && lane + above < lim) {
        sl[lane + above] = L;
        si[lane + above] = I;
    }
    __syncwarp();
    bool bad = false;
    if (lane + 1 < lim) {
        const unsigned a = float_order_bits(sl[lane]), b = float_order_bits(sl[lane + 1]);
        bad = (si[lane] | si[lane + 1]) < 0 && b - a + kKeyUlps <= 2u * kKeyUlps;
    }
    const bool ok = !__any_sync(FULL, bad);
    __syncwarp();  // the reads above before any lane's next write of sl / si (memory order, not just a vote)
    return ok;
}

// One pixel's K'-nearest selection (warp-wide) over a depth-ordered candidate
// list (or, overflow, every kernel): lanes stride the list 32 candidates at a
// time; box test (one 16-byte load), FP32 q classification and depth key for
// the eligible lanes; the K' nearest kept warp-distributed and sorted (lane s
// holds the s-th nearest) as FP32 rank keys + kernel ids; eligible candidates
// merged per batch (merge_batch, or ranks from ballots with exact-trace
// tie-breaks). Writes topk / count of the pixel; returns the count.
__device__ __forceinline__ int select_pixel(const FwdParams& p, const unsigned long long* list, int end, bool overflow,
                                            const double* d, float u, float v, float nrm, int i, int j,
                                            const QClass& qc, bool exact_only, float* sl, int* si, int lane) {
    const unsigned FULL = 0xffffffffu;
    const int kp = p.sel.kp;
    const Rec64* rec64 = p.rec64;
    const double log_eta = p.sel.log_eta;
    const bool early = !overflow;  // the list is ordered by its depth bound
    const int start = 0;
    const long long pix = (long long)i * p.cam.W + j;
    const float fi = (float)i, fj = (float)j;

    float L = INFINITY;  // lane s < n: rank key of the s-th nearest
    int I = 0x7fffffff;
    int n = 0;
    float worst = INFINITY;  // key of lane kp-1 once full (warp-uniform)

    for (int base = start; base < end; base += 32) {
        const int e = base + lane;
        const bool valid = e < end;
        const int k = overflow ? (valid ? e : 0) : (int)(list[valid ? e : 0] & 0xffffffffu);
        // early exit: lists are sorted by zmin <= l; the batch's first zmin bounds the rest
        if (early) {
            const float zmin0 = float_from_order_bits((uint32_t)(list[base] >> 32));
            if (zmin0 > worst + 2.0f * kKeyClose * fabsf(worst)) break;
        }
        const float4* rp = reinterpret_cast<const float4*>(p.rec32 + k);
        const float4 box = __ldg(rp);        // top, bottom, left, right
        const float4 zrec = __ldg(rp + 1);   // zmin, z, ci_frac, cj_frac
        // zmin <= l for any kernel that can pass eta: a candidate whose bound is
        // past the worst kept key cannot enter the full list (skip the tests)
        const bool in_box = valid && fi >= box.x && fi <= box.y && fj >= box.z && fj <= box.w &&
                            !(zrec.x > worst + 2.0f * kKeyClose * fabsf(worst));
        int cls = 0;
        float lk = INFINITY;
        if (in_box) {
            Rec32 r;
            r.zmin = zrec.x;
            r.z = zrec.y;
            r.ci_frac = zrec.z;
            r.cj_frac = zrec.w;
            const float4 c2 = __ldg(rp + 2), c3 = __ldg(rp + 3);
            r.ci_int = __float_as_int(c2.x);
            r.cj_int = __float_as_int(c2.y);
            r.s00 = c2.z;
            r.s01 = c2.w;
            r.s02 = c3.x;
            r.s11 = c3.y;
            r.s12 = c3.z;
            r.s22 = c3.w;
            cls = classify_key(r, i, j, u, v, nrm, qc, &lk);
        }
        if (cls != 0) {
            if (exact_only || cls == 1) {
                const double dr[3] = {d[0], d[1], d[2]};
                const Traced64 t = trace_exact(dr, rec64[k]);
                if (t.q > log_eta) {  // fine_select threshold (tracer.cpp:117-118)
                    lk = (float)t.l;
                } else {
                    cls = 0;
                }
            }
            // cannot enter a full list
            if (cls != 0 && lk > worst + 2.0f * kKeyClose * fabsf(worst)) cls = 0;
        }
        const unsigned elig = __ballot_sync(FULL, cls != 0);
        if (elig == 0) continue;
        const bool me = (elig >> lane) & 1u;
        const int m = __popc(elig);
        bool merged = false;
        if (m >= GVR_SEL_BATCH_MIN) merged = merge_batch(L, I, n, lk, k, me, m, kp, lane, sl, si);
        if (!merged) {
        // ranks: for each eligible candidate (broadcast), the kept keys and the
        // other candidates smaller than it; kept entries count the candidates
        // that precede them.
        int shift = 0, mypos = 0;
        unsigned pend = elig;
        while (pend) {
            const int src = __ffs(pend) - 1;
            pend &= pend - 1;
            const float bl = __shfl_sync(FULL, lk, src);
            const int bi = __shfl_sync(FULL, k, src);
            const bool in_ex = lane < n, in_c = me && lane != src;
            bool ex_lt = in_ex && L < bl;
            bool c_lt = in_c && lk < bl;
            const bool ex_close = in_ex && keyf_close(L, bl);
            const bool c_close = in_c && keyf_close(lk, bl);
            if (__any_sync(FULL, ex_close || c_close)) {  // rare: decide on the exact trace
                if (ex_close) ex_lt = exact_less(I, bi, d, rec64);
                if (c_close) c_lt = exact_less(k, bi, d, rec64);
            }
            const int pos = __popc(__ballot_sync(FULL, ex_lt)) + __popc(__ballot_sync(FULL, c_lt));
            if (lane == src) mypos = pos;
            if (in_ex && !ex_lt) ++shift;
        }
        // scatter into the merged order, keep the first kp
        if (lane < n && lane + shift < kp) {
            sl[lane + shift] = L;
            si[lane + shift] = I;
        }
        if (me && mypos < kp) {
            sl[mypos] = lk;
            si[mypos] = k;
        }
        }
        __syncwarp();
        n = min(n + m, kp);
        L = lane < n ? sl[lane] : INFINITY;
        I = lane < n ? (si[lane] & 0x7fffffff) : 0x7fffffff;
        __syncwarp();
        if (n == kp) worst = __shfl_sync(FULL, L, kp - 1);
    }
    if (lane < n) p.topk[pix * kp + lane] = I;  // exact (l, idx) order
    if (lane == 0) p.count[pix] = n;
    return n;
}

// K3a selection, warp-per-pixel form (K' <= 32). CTA = one 8x8 tile, 8 warps;
// warp w handles pixels w, w+8, ... of the tile. Lanes stride the tile's list
// 32 candidates at a time: box test (one 16-byte load), FP32 q classification
// and fast l for the eligible lanes, all lane-parallel. The K' nearest live
// warp-distributed and sorted (lane s holds the s-th nearest) as FP32 rank keys
// + kernel ids; a batch's eligible candidates are merged in one step: ranks
// from ballots, then one scatter through a per-warp shared-memory buffer. Any
// comparison between keys within the FP32 bound is decided on the exact trace,
// so the kept set is exactly the reference's.
template <int KMAX>
__global__ void __launch_bounds__(256 / GVR_SEL_SPLIT, GVR_SEL_MINB) select_warp_kernel(FwdParams p) {
    constexpr int TILE = 8;
    __shared__ float sh_l[8][64];
    __shared__ int sh_i[8][64];
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    // GVR_SEL_SPLIT CTAs per tile, each 8 / GVR_SEL_SPLIT warps (2x4 sub-blocks)
    launch_dependents();  // the blend may fill the SMs this grid's tail leaves idle
    if ((int)(blockIdx.x / GVR_SEL_SPLIT) >= *p.n_order) return;
    __shared__ long long sh_t0;  // the CTA's start (cost hint, profiling hook; kept out of registers)
    if (threadIdx.x == 0) sh_t0 = clock64();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sb = (blockIdx.x % GVR_SEL_SPLIT) * (8 / GVR_SEL_SPLIT) + warp;  // sub-block of the tile
    const unsigned FULL = 0xffffffffu;
    const int tile = p.tile_order[blockIdx.x / GVR_SEL_SPLIT];
    const int smem_cap = kSelListSmem;  // shared-memory layout; p.list_smem decides where a list is sorted
    const unsigned long long* tl = keys;
    // staged through the per-warp list area (free until the compaction below)
    const int listed = load_sorted_list(p, tile, keys, p.list_smem, &tl, keys + smem_cap);
    const bool overflow = listed < 0;  // stream every kernel, unsorted, no early exit
    // Each warp owns a 2x4-pixel sub-block of the tile and first compacts the
    // tile list to the entries whose screen box meets the sub-block (stable, so
    // the depth order survives): its pixels then scan ~half the list. Lists
    // longer than kWarpListCap stay on the tile list.
    const int sr0 = (tile / p.tiles_x) * TILE + (sb >> 1) * 2;
    const int sc0 = (tile % p.tiles_x) * TILE + (sb & 1) * 4;
    unsigned long long* wlist = keys + smem_cap + warp * kWarpListCap;
    const unsigned long long* list = tl;
    int end = overflow ? p.K : listed;
    if (!overflow) {
        const float fr0 = (float)sr0, fr1 = (float)(sr0 + 1), fc0 = (float)sc0, fc1 = (float)(sc0 + 3);
        int cnt = 0;
        // GVR_SEL_CUNROLL batches per step: their boxes' loads are in flight together
        for (int base = 0; base < listed && cnt <= kWarpListCap; base += 32 * GVR_SEL_CUNROLL) {
            unsigned long long key[GVR_SEL_CUNROLL];
            float4 box[GVR_SEL_CUNROLL];
#pragma unroll
            for (int h = 0; h < GVR_SEL_CUNROLL; ++h) {
                key[h] = 0ull;
                const int e = base + 32 * h + lane;
                if (e < listed) {
                    key[h] = tl[e];
                    box[h] = __ldg(reinterpret_cast<const float4*>(p.rec32 + (int)(key[h] & 0xffffffffu)));
                }
            }
#pragma unroll
            for (int h = 0; h < GVR_SEL_CUNROLL; ++h) {
                const int e = base + 32 * h + lane;
                const bool hit = e < listed && box[h].x <= fr1 && box[h].y >= fr0 && box[h].z <= fc1 &&
                                 box[h].w >= fc0;
                const unsigned b = __ballot_sync(FULL, hit);
                const int off = cnt + __popc(b & ((1u << lane) - 1u));
                if (hit && off < kWarpListCap) wlist[off] = key[h];
                cnt += __popc(b);
            }
        }
        __syncwarp();
        if (cnt <= kWarpListCap) {
            list = wlist;
            end = cnt;
        }
    }
    // dynamic pixel queue: the CTA's 64 pixels, heaviest sub-blocks first, are
    // pulled by whichever warp is free (the CTA ends with its last pixel, not
    // with its slowest warp)
    constexpr int NSB = 8 / GVR_SEL_SPLIT;  // sub-blocks (= warps) of this CTA
    __shared__ int sh_end[NSB], sh_sbo[NSB], sh_next;
    __shared__ int2 sh_tile_rc;  // the tile's first pixel row / column
    if (threadIdx.x == 0) sh_tile_rc = make_int2(sr0 - (sb >> 1) * 2, sc0 - (sb & 1) * 4);
    if (lane == 0) sh_end[warp] = list == wlist ? end : -1;
    if (threadIdx.x == 0) sh_next = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int a = 0; a < NSB; ++a) sh_sbo[a] = a;
        for (int a = 1; a < NSB; ++a) {  // insertion sort by list length, descending (-1 = tile list: longest)
            const int v = sh_sbo[a];
            const int ev = sh_end[v] < 0 ? 0x7fffffff : sh_end[v];
            int b = a - 1;
            while (b >= 0 && (sh_end[sh_sbo[b]] < 0 ? 0x7fffffff : sh_end[sh_sbo[b]]) < ev) {
                sh_sbo[b + 1] = sh_sbo[b];
                --b;
            }
            sh_sbo[b + 1] = v;
        }
    }
    // the tile's 64 rays (FP64, exact path) and their FP32 image-plane
    // coordinates and |dt| (pre-filter and depth keys), once per CTA
    __shared__ double sh_ray[64][3];
    __shared__ float4 sh_uvn[64];
    for (int q = threadIdx.x; q < 64; q += blockDim.x) {
        const int ri = (tile / p.tiles_x) * TILE + q / TILE, rj = (tile % p.tiles_x) * TILE + q % TILE;
        if (ri < p.cam.H && rj < p.cam.W) {
            double d[3];
            pixel_ray(p.cam, ri, rj, d);
            sh_ray[q][0] = d[0];
            sh_ray[q][1] = d[1];
            sh_ray[q][2] = d[2];
            const double u = xdiv(xsub((double)ri, p.cam.oy), p.cam.focal);
            const double v = xdiv(xsub((double)rj, p.cam.ox), p.cam.focal);
            sh_uvn[q] = make_float4((float)u, (float)v, (float)sqrt(u * u + v * v + 1.0), 0.0f);
        }
    }
    __syncthreads();
    const QClass& qc = p.qc;  // kernel parameter space: no registers
    const bool exact_only = p.exact_only != 0;

    for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(&sh_next, 1);
        item = __shfl_sync(FULL, item, 0);
        if (item >= NSB * 8) break;
        const int pw = sh_sbo[item >> 3], px = item & 7;  // owning warp, pixel of its sub-block
        const int psb = (blockIdx.x % GVR_SEL_SPLIT) * NSB + pw;
        const int psr = sh_tile_rc.x + (psb >> 1) * 2;  // (no per-item division)
        const int psc = sh_tile_rc.y + (psb & 1) * 4;
        const int i = psr + (px >> 2);
        const int j = psc + (px & 3);
        const int pe = sh_end[pw];
        list = pe >= 0 ? keys + smem_cap + pw * kWarpListCap : tl;
        end = pe >= 0 ? pe : (overflow ? p.K : listed);
        if (i >= p.cam.H || j >= p.cam.W) continue;  // warp-uniform
        const int q = ((psb >> 1) * 2 + (px >> 2)) * TILE + (psb & 1) * 4 + (px & 3);  // pixel within the tile
        const double* d = sh_ray[q];  // read only on the exact path
        const float4 uvn = sh_uvn[q];
        const float u = uvn.x, v = uvn.y, nrm = uvn.z;
        select_pixel(p, list, end, overflow, d, u, v, nrm, i, j, qc, exact_only, sh_l[warp], sh_i[warp], lane);
    }
    if (p.tile_done || p.tile_cycles || p.tile_hint) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const long long dt = clock64() - sh_t0;  // the CTA's duration (its slowest warp)
            if (p.tile_cycles)  // profiling hook
                atomicAdd(reinterpret_cast<unsigned long long*>(p.tile_cycles + tile), (unsigned long long)dt);
            if (p.tile_hint) p.tile_hint[tile] = (unsigned)min(max(dt, 1ll), 0xffffffffll);
            if (p.tile_done) red_add_release_gpu(p.tile_done + tile, 1u);  // one count per split CTA
        }
    }
}

// The pixel's bit in each selected kernel's (kernel, tile) mask: the backward's
// per-kernel record order (order-independent OR). Entries s = sub, sub + 4, ...
__device__ __forceinline__ void mark_selection(const FwdParams& p, const int* b_slot, int n, int sub, int g, int np,
                                               int i, int j) {
    for (int s = sub; s < n; s += 4) {
        const int slot = b_slot[s * np + g];
        if (slot >= 0) atomicOr(p.masks + slot, 1ull << ((i % 8) * 8 + j % 8));
    }
}

// K3b closed-form blend (blender.cpp:27-53, 98-128). CTA = one 8x8 tile with
// 4 threads per pixel (256 threads): entries are re-traced (exact FP64) and the
// O(n^2) transmittance sums split 4 ways; the ordered attribute/depth sums are
// then done by one thread per pixel so that image == sum_k W_k attr_k exactly
// in ascending (l, idx) order.
//   W_k = exp(-tau sum_m e^{q_m} Phi((l_k - l_m)/sigma_m)) e^{q_k}
// The sum is accumulated in FP64 and T(l_k) is taped for the backward.
// Blend staging slot: the traced l with the FP32 peak and 1/sigma; after the
// sort the first 8 bytes become the float pair (hi, lo) of l - l_0, so the pair
// loop reads everything it needs about entry m with one 16-byte load.
#ifndef GVR_BLEND_STAGE
#define GVR_BLEND_STAGE 1
#endif
// per-warp record stage of the blend: 32 records at a 144-byte stride (9 x 16 B:
// the 8 lanes of a quarter-warp reading 16 bytes each hit distinct banks)
constexpr int kStageRecU4 = 9;
constexpr size_t kBlendStageBytes = GVR_BLEND_STAGE ? (256 / GVR_BLEND_SPLIT) * 16 * kStageRecU4 : 0;
struct __align__(16) BlendSlot {
    double l;
    float pk, is;
};

template <int KMAX>
__global__ void __launch_bounds__(256 / GVR_BLEND_SPLIT, GVR_BLEND_MINB) blend_kernel(FwdParams p) {
    constexpr int TILE = 8, NP = 64 / GVR_BLEND_SPLIT, PER = (KMAX + 3) / 4;
    extern __shared__ __align__(16) unsigned char smem[];
    BlendSlot* b_s = reinterpret_cast<BlendSlot*>(smem);  // [slot][pixel]
    const float4* b_q = reinterpret_cast<const float4*>(smem);  // {hi, lo, pk, is} after the conversion
    double* b_w = reinterpret_cast<double*>(b_s + KMAX * NP);  // W_k
    int* b_id = reinterpret_cast<int*>(b_w + KMAX * NP);
    int* b_slot = b_id + KMAX * NP;  // the entry's (kernel, tile) mask slot, -1: none (selection order)

    // the order counts and this CTA's tile are loaded together (the order array
    // holds every tile, so the read is in bounds before the count check)
    const int bt = (int)(blockIdx.x / GVR_BLEND_SPLIT);
    const int n_blend = *p.n_order_blend, n_sel = *p.n_order;
    const int tile = p.tile_order_blend[bt];
    if (bt >= n_blend) return;
    const int g = threadIdx.x >> 2, sub = threadIdx.x & 3;
    if (p.tile_done && bt < n_sel) {
        // started early (programmatic dependent of the selection): wait for this tile only
        if (threadIdx.x == 0) {
            // bounded: a selection that never publishes (a bug) must fail the launch, not hang the device
            for (unsigned spin = 0; ld_acquire_gpu(p.tile_done + tile) < (unsigned)GVR_SEL_SPLIT; ++spin) {
                if (spin > (1u << 26)) __trap();
                __nanosleep(GVR_PDL_SLEEP_NS);
            }
        }
        __syncthreads();
    }
    const int gp = (blockIdx.x % GVR_BLEND_SPLIT) * NP + g;  // pixel within the tile
    const int i = (tile / p.tiles_x) * TILE + gp / TILE;
    const int j = (tile % p.tiles_x) * TILE + gp % TILE;
    const bool inside = i < p.cam.H && j < p.cam.W;
    const long long pix = (long long)i * p.cam.W + j;
    const int kp = p.sel.kp;
    // tiles after the selected ones in the order (other shards, empty lists) are
    // cleared; a selected tile has a count for every pixel
    const bool visited = bt < n_sel;
    // the pixel's whole top-K row is loaded with its count (one dependent hop
    // fewer before the record loads; slots past the count are never used)
    int ids[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int s = sub + 4 * q;
        ids[q] = inside && visited && s < kp ? __ldcg(p.topk + pix * kp + s) : 0;
    }
    const int n = inside && visited ? p.count[pix] : 0;
    double d[3];
    double peak_part = 0.0;
    // one traced entry: FP64 peak, taped l / 1/sigma, id and the kernel's mask
    // slot for this tile
    auto trace_entry = [&](int s, int k, const Rec64& r) {
        const Traced64 t = trace_fast(d, r);
        const double pk = exp(t.q);
        b_w[s * NP + g] = pk;  // FP64 peak until W overwrites it (alpha sum, after the sort)
        if (p.presorted) p.ent_a[pix * kp + s] = t.a;
        BlendSlot v;
        v.l = t.l;  // l for now; relative to the nearest after the sort
        v.pk = (float)pk;
        v.is = (float)sqrt(t.a);  // 1/sigma
        b_s[s * NP + g] = v;
        b_id[s * NP + g] = k;
        const int4 ki = p.kinfo[k];
        b_slot[s * NP + g] = ki.x >= 0 ? ki.x + (i / 8 - (ki.y >> 16)) * ki.z + (j / 8 - (ki.y & 0xffff)) : -1;
    };
#if GVR_BLEND_STAGE
    {
        // The records are staged per warp through shared memory, one round per
        // entry slot sub + 4q: the warp copies its lanes' 32 records with
        // coalesced 16-byte loads (8 lanes per 128-byte record, 4 records per
        // instruction) instead of each lane reading its own record (32 lines
        // per load instruction: the L1 wavefronts were the blend's busiest
        // unit). All lanes of the CTA are present here (empty pixels included).
        const unsigned FULL = 0xffffffffu;
        const int lane = threadIdx.x & 31;
        uint4* st = reinterpret_cast<uint4*>(smem + 32 * KMAX * NP) + (threadIdx.x >> 5) * (32 * kStageRecU4);
        const int qmax = (int)__reduce_max_sync(FULL, (unsigned)((n + 3) >> 2));
        if (n > 0) pixel_ray(p.cam, i, j, d);
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            if (q >= qmax) break;  // warp-uniform
            const int s = sub + 4 * q;
            const int myid = s < n ? ids[q] : -1;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int src = (lane >> 3) + 4 * c;
                const int kid = __shfl_sync(FULL, myid, src);
                if (kid >= 0)
                    st[src * kStageRecU4 + (lane & 7)] = __ldg(reinterpret_cast<const uint4*>(p.rec64 + kid) + (lane & 7));
            }
            __syncwarp();
            if (s < n) trace_entry(s, ids[q], *reinterpret_cast<const Rec64*>(st + lane * kStageRecU4));
            __syncwarp();  // the stage is rewritten by the next round
        }
    }
#endif
    if (n == 0) {
        if (inside && sub == 0) {
            for (int c = 0; c < p.Dc; ++c) p.image[pix * p.Dc + c] = 0.0;
            p.alpha[pix] = 0.0;
            p.depth[pix] = 0.0;
            if (!visited) p.count[pix] = 0;
        }
        return;  // the 4 threads of a pixel leave together
    }
    const unsigned grp = 0xfu << (threadIdx.x & 28);  // the pixel's 4 lanes
#if !GVR_BLEND_STAGE
    pixel_ray(p.cam, i, j, d);
#pragma unroll
    for (int q = 0; q < PER; ++q)
        if (sub + 4 * q < n) trace_entry(sub + 4 * q, ids[q], p.rec64[ids[q]]);
#endif
    __syncwarp(grp);
    if (sub == 0 && !p.presorted) {
        // ascending (l, idx) of fine_select (tracer.cpp:119-122): insertion sort;
        // keys closer than the fast-trace error are compared on exact l
        for (int s = 1; s < n; ++s) {
            BlendSlot vs = b_s[s * NP + g];
            int is = b_id[s * NP + g];
            const double ws = b_w[s * NP + g];
            int t = s - 1;
            while (t >= 0) {
                BlendSlot vt = b_s[t * NP + g];
                int it = b_id[t * NP + g];
                const bool less = key_less(vs.l, is, vt.l, it, d, p.rec64);
                b_s[t * NP + g] = vt;  // possibly upgraded to exact
                b_id[t * NP + g] = it;
                if (!less) break;
                b_s[(t + 1) * NP + g] = vt;
                b_id[(t + 1) * NP + g] = it;
                b_w[(t + 1) * NP + g] = b_w[t * NP + g];
                --t;
            }
            b_s[(t + 1) * NP + g] = vs;
            b_id[(t + 1) * NP + g] = is;
            b_w[(t + 1) * NP + g] = ws;
        }
    }
    __syncwarp(grp);
    // sum of peaks in the (exact) entry order: deterministic whatever order the
    // selection produced the set in
    for (int s = sub; s < n; s += 4) peak_part += b_w[s * NP + g];
    peak_part += __shfl_xor_sync(grp, peak_part, 1, 4);
    peak_part += __shfl_xor_sync(grp, peak_part, 2, 4);
    const double l0 = b_s[g].l;
    __syncwarp(grp);
    // l_k - l_0 as an unevaluated float pair hi + lo (replaces the double in place):
    // hi_k - hi_m is exact whenever the pair's z is moderate (Sterbenz), so the
    // argument z = (l_k - l_m) / sigma_m keeps ~1e-7 relative accuracy in FP32.
    for (int s = sub; s < n; s += 4) {
        const BlendSlot v = b_s[s * NP + g];
        const double lval = v.l;
        const double dl = lval - l0;
        const float hi = (float)dl;
        reinterpret_cast<float2*>(&b_s[s * NP + g].l)[0] = make_float2(hi, (float)(dl - (double)hi));
        if (!p.presorted) {
            b_id[s * NP + g] &= ~kExact;
            p.topk[pix * kp + s] = b_id[s * NP + g];
            p.ent_a[pix * kp + s] = trace_fast(d, p.rec64[b_id[s * NP + g]]).a;  // the same a, sorted order
        }
        // tape the traced entry for the backward and the sampler
        EntryRec er;
        er.l = lval;
        er.pk = v.pk;
        er.is = v.is;
        p.ent[pix * kp + s] = er;
    }
    __syncwarp(grp);

    if (p.precise) {
        // verification mode (gvr_context_set_precise): every pair term from the
        // exact FP64 trace and erfc, W in FP64 -- the reference's arithmetic
        for (int k = sub; k < n; k += 4) {
            const Traced64 tk = trace_exact(d, p.rec64[b_id[k * NP + g]]);
            double acc = 0.0;
            for (int m = 0; m < n; ++m) {
                const Traced64 tm = trace_exact(d, p.rec64[b_id[m * NP + g]]);
                acc += exp(tm.q) * (0.5 * erfc(-((tk.l - tm.l) / sigma_of(tm.a)) * 0.7071067811865476));
            }
            const double trans = exp(-p.tau * acc);
            const double wd = trans * exp(tk.q);
            p.tape_t[pix * kp + k] = trans;
            b_w[k * NP + g] = wd;
            if (p.topk_w) p.topk_w[pix * kp + k] = wd;
        }
    }
    for (int k = sub; k < n && !p.precise; k += 4) {
        const float4 hk = b_q[k * NP + g];
        // sum_m e^{q_m} Phi(z_km): non-negative FP32 terms, Kahan-compensated
        // (error ~2^-24 of the sum, below the 6e-8 of the Phi approximation)
        float sum = 0.0f, comp = 0.0f;
        for (int m = 0; m < n; ++m) {
            const float4 hm = b_q[m * NP + g];  // {hi, lo, pk, 1/sigma}
            const float z = ((hk.x - hm.x) + (hk.y - hm.y)) * hm.w;
            const float y = fmaf(hm.z, fast_normal_cdf(z), -comp);
            const float t = sum + y;
            comp = (t - sum) - y;
            sum = t;
        }
        const double acc = (double)sum - (double)comp;
        const double trans = exp(-p.tau * acc);
        const double wd = trans * (double)hk.z;
        p.tape_t[pix * kp + k] = trans;
        b_w[k * NP + g] = wd;
        if (p.topk_w) p.topk_w[pix * kp + k] = wd;
    }
    __syncwarp(grp);
    const double alpha = 1.0 - exp(-p.tau * peak_part);
    if (p.D <= 3) {
        // ordered sums, one thread per output, products loaded 4 ahead:
        // image[c] = sum_k W_k attr_k[c] exactly in ascending (l, idx) order
        if (sub < p.D) {
            double img = 0.0;
            int k = 0;
            for (; k + 4 <= n; k += 4) {
                double a[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = p.attr[(long long)p.D * b_id[(k + u) * NP + g] + sub];
#pragma unroll
                for (int u = 0; u < 4; ++u) img = xadd(img, xmul(b_w[(k + u) * NP + g], a[u]));
            }
            for (; k < n; ++k) img = xadd(img, xmul(b_w[k * NP + g], p.attr[(long long)p.D * b_id[k * NP + g] + sub]));
            p.image[pix * p.Dc + sub] = img;
            if (!isfinite(img)) atomicExch(p.nonfinite, 1);
        } else if (sub == 3) {
            if (p.D == 0) p.image[pix * p.Dc] = 0.0;
            double wsum = 0.0, wld = 0.0;
            for (int k = 0; k < n; ++k) {
                const double wd = b_w[k * NP + g];
                wsum += wd;
                const float4 h = b_q[k * NP + g];
                wld += wd * (l0 + ((double)h.x + (double)h.y));
            }
            const double depth = wsum > 1e-12 ? wld / wsum : 0.0;
            p.alpha[pix] = alpha;
            p.depth[pix] = depth;
            if (!isfinite(alpha) || !isfinite(depth) || !isfinite(wsum)) atomicExch(p.nonfinite, 1);
        }
        mark_selection(p, b_slot, n, sub, g, NP, i, j);
        return;
    }
    mark_selection(p, b_slot, n, sub, g, NP, i, j);
    if (sub != 0) return;
    double wsum = 0.0, wld = 0.0;
    for (int k = 0; k < n; ++k) {
        const double wd = b_w[k * NP + g];
        const int kid = b_id[k * NP + g];
        for (int c = 0; c < p.D; ++c) {
            const long long o = pix * p.Dc + c;
            p.image[o] = xadd(k == 0 ? 0.0 : p.image[o], xmul(wd, p.attr[(long long)p.D * kid + c]));
        }
        wsum += wd;
        const float4 h = b_q[k * NP + g];
        wld += wd * (l0 + ((double)h.x + (double)h.y));
    }
    const double depth = wsum > 1e-12 ? wld / wsum : 0.0;
    p.alpha[pix] = alpha;
    p.depth[pix] = depth;
    bool bad = !isfinite(alpha) || !isfinite(depth) || !isfinite(wsum);
    for (int c = 0; c < p.D && n > 0; ++c) bad = bad || !isfinite(p.image[pix * p.Dc + c]);
    if (bad) atomicExch(p.nonfinite, 1);
}

// Tile-list layout (blockDim.x == 1024): exclusive scan of the per-tile counts
// in tile order into pool offsets. Lists that would end past pool_cap get
// offset -1 (streamed by the selection, counted as overflow). stats: [0] total
// entries, [1] longest list, [2] overflowed tiles, [3] lists longer than
// smem_cap (sorted in the global sorted pool).
__device__ void list_offsets(int tiles, const int* __restrict__ count, int* __restrict__ tile_off, int pool_cap,
                             int smem_cap, int* __restrict__ stats) {
    __shared__ long long s_warp[32];
    __shared__ int s_max, s_over, s_long;
    if (threadIdx.x == 0) s_max = s_over = s_long = 0;
    const int chunk = (tiles + 1023) / 1024;
    const int t0 = min(tiles, (int)threadIdx.x * chunk), t1 = min(tiles, t0 + chunk);
    long long run = 0;
    int mx = 0;
    for (int t = t0; t < t1; ++t) {
        run += count[t];
        mx = max(mx, count[t]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (lane == 0) atomicMax(&s_max, mx);
    if (warp == 0) {
        long long w = s_warp[lane], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_warp[lane] = wi - w;  // exclusive
        if (lane == 31) stats[0] = (int)min(wi, (long long)0x7fffffff);
    }
    __syncthreads();
    long long off = s_warp[warp] + incl - run;
    int over = 0, lng = 0;
    for (int t = t0; t < t1; ++t) {
        const int c = count[t];
        const bool fits = c > 0 && off + c <= (long long)pool_cap;
        tile_off[t] = fits ? (int)off : -1;
        over += c > 0 && !fits;
        lng += fits && c > smem_cap;
        off += c;
    }
    if (over) atomicAdd(&s_over, over);
    if (lng) atomicAdd(&s_long, lng);
    __syncthreads();
    if (threadIdx.x == 0) {
        stats[1] = s_max;
        stats[2] = s_over;
        stats[3] = s_long;
    }
}

constexpr int kOrderSmemTiles = 16384;  // 6 B of shared memory per tile (96 KB)

// Longest-processing-time-first order of tiles (single-CTA counting sort over
// log-spaced cost buckets, descending). Zero-cost tiles and tiles of other
// shards (t % nshards != shard) are dropped; *n_out receives the number kept.
// Cost = icost[t] (list length); with a hint (the selection cycles
// of the previous render of the same view, tile_hint) the listed tiles are
// ordered by it instead. With tile_off, the tile-list offsets are laid out
// first (list_offsets; icost = the list lengths).
__global__ void __launch_bounds__(1024) order_tiles_kernel(int tiles, const int* __restrict__ icost,
                                                           int* __restrict__ order,
                                                           int* __restrict__ n_out, int shard, int nshards,
                                                           int* __restrict__ n_all_out, int* __restrict__ tile_off = nullptr,
                                                           int pool_cap = 0, int smem_cap = 0,
                                                           int* __restrict__ stats = nullptr,
                                                           const unsigned* __restrict__ hint = nullptr) {
    __shared__ int hist[256];
    __shared__ int offs[256];
    __shared__ int s_tail;
    // up to kOrderSmemTiles tiles: counts and buckets read from global memory once
    // (all loads of a thread in flight together) into shared memory for every pass
    extern __shared__ int s_dyn[];
    const bool staged = tiles <= kOrderSmemTiles;
    int* s_cnt = s_dyn;
    short* s_bkt = reinterpret_cast<short*>(s_dyn + (staged ? tiles : 0));
    auto bucket_from = [&](int t, int cnt, unsigned h) -> int {
        if (t % nshards != shard) return -1;  // tile owned by another rank (C4 tile sharding)
        float c = (float)cnt;
        if (!(c > 0.0f)) return -1;
        if (hint) c = h > 0u ? (float)h : 100.0f * c;  // cycles (a tile new to the view: ~100 / entry)
        const int b = (int)(__log2f(c + 1.0f) * 8.0f);
        return 255 - min(b, 255);  // descending cost
    };
    if (staged) {
#pragma unroll 4
        for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
            const int c = icost[t];
            const unsigned h = hint ? hint[t] : 0u;
            s_cnt[t] = c;
            s_bkt[t] = (short)bucket_from(t, c, h);
        }
        __syncthreads();
    }
    auto bucket_of = [&](int t) -> int {
        return staged ? (int)s_bkt[t] : bucket_from(t, icost[t], hint ? hint[t] : 0u);
    };
    if (tile_off) list_offsets(tiles, staged ? s_cnt : icost, tile_off, pool_cap, smem_cap, stats);
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
        const int b = bucket_of(t);
        if (b >= 0) atomicAdd(&hist[b], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp scan over the 256 buckets
        int vals[8], run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            vals[q] = hist[threadIdx.x * 8 + q];
            run += vals[q];
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (threadIdx.x >= o) incl += y;
        }
        int base = incl - run;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            offs[threadIdx.x * 8 + q] = base;
            base += vals[q];
        }
        if (threadIdx.x == 31) {
            *n_out = incl;
            s_tail = incl;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
        const int b = bucket_of(t);
        if (b >= 0) order[atomicAdd(&offs[b], 1)] = t;
    }
    if (n_all_out) {  // then every other tile (the blend clears them): order holds all tiles
        for (int t = threadIdx.x; t < tiles; t += blockDim.x)
            if (bucket_of(t) < 0) order[atomicAdd(&s_tail, 1)] = t;
        __syncthreads();
        if (threadIdx.x == 0) *n_all_out = s_tail;
    }
}

}  // namespace gvrk
