// Fused explicit-Euler step of the layered field (sm_100a): active-set
// stepping on the hybrid field layout.
//
// One step replaces the reference pipeline of field.step
// (reference pkg/src/fieldtess/field.py:198-286):
//
//   Lt = PHI L^T            spgemm_numeric      _kernels.py:26-62
//   interest skeleton       skeleton_count/fill _kernels.py:96-150
//   PHI^, Lt^ expansion     expand_kernel       _kernels.py:153-176
//   Euler update + clamp    update_kernel       _kernels.py:179-238
//   normalise + compact     column_sums_counts, normalize_compact
//                                               _kernels.py:241-282
//
// Column j of the new field is a function of the columns u in L^T(:, j)
// (its closed one-ring) only.  So if none of them changed in the previous
// step, column j does not change either, and the ping-pong target buffer --
// which holds column j of two steps ago, equal to its current value -- is
// already correct.  Every kernel that writes a column compares it with its
// input; a changed column stamps its one-ring "active" for the next step
// (byte stamps, the step sequence number mod 256: stale stamps only add
// work, they never drop any).  A step is then
//
//   prep_kernel    compacts this step's stamps into the active list (or, on
//                  a full step, lets the column kernels walk every column);
//   band_kernel    one lane per active column: the neighbours' row
//                  signatures classify it; a single-row neighbourhood takes
//                  the exact closed form, a two-row one the straight-line
//                  two-row update (process_two); anything wider is listed;
//   wide3_kernel   the listed columns, one lane each: up to three rows and
//                  three entries per neighbour (process_window<3>); wider
//                  ones are listed again;
//   wide4_kernel   (when they are many) those, one lane each: up to four
//                  rows and four entries per neighbour (process_window<4>);
//   wide_kernel    the rest, one warp each: the neighbourhood staged in
//                  shared memory and ranked by row, Lt and the column sums
//                  taken in the reference's order; beyond the staging
//                  capacity the column is listed for the deep pass;
//   finalize       the deep pass (the exact windowed algorithm from global
//                  memory, one lane per listed column; rare), then the
//                  statistics record, status, convergence, next-step mode.
//
// Statistics are order-independent -- integer nnz / skeleton counts, a max,
// and the base mass in exact fixed point (ft_common.cuh fx_split) -- so an
// active step updates the running totals by the changes of its active
// columns and every kernel folds its columns in with CTA-level atomics; the
// result is deterministic and equal to the full recomputation.
//
// Active-set stepping needs the pattern of L^T to be symmetric (column j
// is read by exactly the columns it reads); the host asserts it with
// FT_LAP_SYMMETRIC, otherwise (and in a partitioned domain) every step is a
// full step.  A full step also runs after ft_tiled_from_csc and when the
// target buffer's pool is half used (pool columns recycle their own range in
// place when it is large enough, new ones take fresh entries; a full step
// re-packs the pool).
//
// EXACT mode (double storage) replays the reference arithmetic operation by
// operation (ft_arith.cuh); FAST mode stores PHI in float and does all
// arithmetic in double, in the same order.

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>

#include "ft_arith.cuh"
#include "ft_common.cuh"

namespace ft {

// exact 1.0 / n for n = 0..32 (host IEEE division; entry 0 unused)
__constant__ double c_recip[33];

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start before its
// predecessor in the stream has finished; it waits here, before touching
// anything.  A no-op for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ T vload(const T* p) { return *(volatile const T*)p; }

// 1-D bulk copies (TMA, cp.async.bulk) global -> shared, completed on an
// mbarrier with a transaction count
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to the async proxy
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)), "r"(phase) : "memory");
}

constexpr unsigned int kFull = 0xffffffffu;

struct StepParams {
    int n_v;             // owned columns (the whole field outside domain mode)
    int j_base;          // global index of the first owned column
    const int* __restrict__ lap_ptr;
    const int* __restrict__ lap_idx;
    const void* __restrict__ lap_val;
    const int4* __restrict__ lap_pack;  // FT_LAP_PACKED: int16 deltas u - j, 8 per column
    HybIn in;
    HybOut out;
    long long cap;       // pool entries the step may use
    int out_id;          // which pool bump pointer (hybrid buffer 0 / 1)
    int track;           // active-set stepping (symmetric L^T pattern, not a domain)
    int check_done;
    int force_check;     // FT_LAP_CHECK_FINITE: check input values for NaN / Inf
    Cp cp;
    Workspace ws;
    const int* report_ids;  // nullable: caller ids of the owned columns (error reports)
    int wide4_min;       // the four-row kernel runs when the three-row kernel leaves at least this many
};

// the step recomputes every column (always without tracking)
__device__ __forceinline__ bool step_is_full(const StepParams& p) {
    return !p.track || vload(&p.ws.ctl->full) != 0;
}

template <typename T>
__device__ __forceinline__ double ldv(const void* p, long long i) {
    return (double)__ldg(((const T*)p) + i);
}

// bitwise equality of two values as stored (T)
template <typename T>
__device__ __forceinline__ bool same_bits(double a, double b);
template <>
__device__ __forceinline__ bool same_bits<double>(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
}
template <>
__device__ __forceinline__ bool same_bits<float>(double a, double b) {
    return __float_as_int((float)a) == __float_as_int((float)b);
}

__device__ __forceinline__ void report_flags(const VRes& res, int j, const StepParams& p) {
    if (!res.nan && res.bad_phi_row < 0 && res.bad_lt_row < 0) return;
    if (p.report_ids) j = __ldg(&p.report_ids[j - p.j_base]);   // the caller's vertex id
    if (res.nan) atomicMax(&p.ws.ctl->nan_key, (unsigned int)(INT_MAX - j));
    if (res.bad_phi_row >= 0)
        atomicMax(&p.ws.ctl->bad_phi_key, ~(((unsigned long long)j << 32) | (unsigned int)res.bad_phi_row));
    if (res.bad_lt_row >= 0)
        atomicMax(&p.ws.ctl->bad_lt_key, ~(((unsigned long long)j << 32) | (unsigned int)res.bad_lt_row));
}

// ---------------------------------------------------------------------------
// per-CTA statistics: each thread keeps max |delta| and the nnz / skeleton
// changes in registers; base-mass changes (rare once the base layer is
// gone) are folded warp-wise into shared fixed-point limbs.

struct Acc {
    double md;
    int dn, ds;
};

__device__ __forceinline__ void acc_init(Acc& a) { a.md = 0.0; a.dn = 0; a.ds = 0; }

// base-mass change of one column per lane (warp-collective): new - old, or
// new alone on a full step.  The four limb sums are reduced by shuffles
// first, then lane 0 adds them to the CTA's shared limbs; the warp
// reconverges before it leaves (the shared 64-bit add is a CAS loop).
__device__ __forceinline__ void bm_fold(double bm_new, double bm_old, bool full, long long* s_bm) {
    const double o = full ? 0.0 : bm_old;
    const bool nz = __double_as_longlong(bm_new) != __double_as_longlong(o);
    if (!__any_sync(kFull, nz)) return;
    long long a[4], b[4], d[4];
    fx_split(nz ? bm_new : 0.0, a);
    fx_split(nz ? o : 0.0, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        d[k] = a[k] - b[k];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) d[k] += __shfl_xor_sync(kFull, d[k], s);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (d[k] != 0) atomicAdd((unsigned long long*)&s_bm[k], (unsigned long long)d[k]);
    }
    __syncwarp();
}

// CTA reduction of the per-thread accumulators + the shared base-mass limbs
// into the control block (one atomic per counter and CTA)
template <int NT>
__device__ __forceinline__ void acc_flush(Acc a, long long* s_bm, double* s_md, long long* s_cnt, Control* ctl) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a.md = fmax(a.md, __shfl_xor_sync(kFull, a.md, o));
        a.dn += __shfl_xor_sync(kFull, a.dn, o);
        a.ds += __shfl_xor_sync(kFull, a.ds, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_md[w] = a.md;
        s_cnt[2 * w] = a.dn;
        s_cnt[2 * w + 1] = a.ds;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double md = 0.0;
    long long dn = 0, ds = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) {
        md = fmax(md, s_md[k]);
        dn += s_cnt[2 * k];
        ds += s_cnt[2 * k + 1];
    }
    if (md > 0.0) atomicMax(&ctl->maxdelta_bits, (unsigned long long)__double_as_longlong(md));
    if (dn) atomicAdd((unsigned long long*)&ctl->acc_nnz, (unsigned long long)dn);
    if (ds) atomicAdd((unsigned long long*)&ctl->acc_skel, (unsigned long long)ds);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (s_bm[k]) atomicAdd((unsigned long long*)&ctl->acc_bm[k], (unsigned long long)s_bm[k]);
}

// ---------------------------------------------------------------------------
// the L^T column of a vertex

constexpr int kMD = 8;
constexpr int kPackEmpty = -32768;

// The L^T column of j: u[0..n) in stored order (-1 beyond).  PACKED decodes
// the 16-byte row of int16 deltas (u - j; empty slots kPackEmpty; all-empty =
// not packable, read from the CSR); otherwise the CSR.  Returns n, or 0 when
// the column has no entry or more than kMD (-> the wide kernels).
template <bool PACKED>
__device__ __forceinline__ int unpack_lrow(const StepParams& p, int4 pk, int jl, int j, bool active, int (&u)[kMD],
                                           int& q0) {
    int n = 0;
    q0 = 0;
    bool csr = !PACKED;
    if (PACKED) {
        const int w4[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            const int s = (k & 1) ? (w4[k >> 1] >> 16) : ((int)(w4[k >> 1] << 16) >> 16);
            const bool valid = active && s != kPackEmpty;
            u[k] = valid ? j + s : -1;
            n += valid ? 1 : 0;
        }
        csr = active && n == 0;
    }
    if (csr && active) {
        q0 = __ldg(&p.lap_ptr[jl]);
        n = __ldg(&p.lap_ptr[jl + 1]) - q0;
        if (n > kMD || n < 1) n = 0;
#pragma unroll
        for (int k = 0; k < kMD; ++k) u[k] = (k < n) ? __ldg(&p.lap_idx[q0 + k]) : -1;
    } else if (!PACKED) {
#pragma unroll
        for (int k = 0; k < kMD; ++k) u[k] = -1;
    }
    return n;
}

template <typename T, bool UNIFORM>
__device__ __forceinline__ double lap_value(const StepParams& p, int k, int kd, int q0, double invdeg) {
    return UNIFORM ? ((k == kd) ? -1.0 : invdeg) : ldv<T>(p.lap_val, q0 + k);
}

__device__ __forceinline__ double recip_deg(int n) { return n - 1 <= 32 ? c_recip[n - 1] : 1.0 / (double)(n - 1); }

// stamp the closed one-ring of a changed column for the next step
__device__ __forceinline__ void mark_ring(const StepParams& p, const int (&u)[kMD], int n, unsigned char nxt) {
#pragma unroll
    for (int k = 0; k < kMD; ++k)
        if (k < n) p.ws.stamp[u[k]] = nxt;
}

// warp-aggregated push of column j onto a list
__device__ __forceinline__ void list_push(bool push, int j, int* count, int* base, int lane) {
    const unsigned int b = __ballot_sync(kFull, push);
    if (!b) return;
    int q = 0;
    if (lane == 0) q = atomicAdd(count, __popc(b));
    q = __shfl_sync(kFull, q, 0);
    if (push) base[q + __popc(b & ((1u << lane) - 1u))] = j;
}

// warp-staged list: a warp pushes into its own shared buffer (no atomics,
// no barriers) and moves it to the global list with one atomic and a
// coalesced copy when it fills (warp-collective)
struct WarpList {
    int* buf;
    int n;        // entries staged (warp-uniform)
};

__device__ __forceinline__ void wlist_push(bool push, int j, WarpList& l, int lane) {
    const unsigned int b = __ballot_sync(kFull, push);
    if (push) l.buf[l.n + __popc(b & ((1u << lane) - 1u))] = j;
    l.n += __popc(b);
}

__device__ __forceinline__ void wlist_flush(WarpList& l, int* g_count, int* g_list, int lane) {
    __syncwarp();
    if (l.n == 0) return;
    int base = 0;
    if (lane == 0) base = atomicAdd(g_count, l.n);
    base = __shfl_sync(kFull, base, 0);
    for (int k = lane; k < l.n; k += 32) g_list[base + k] = l.buf[k];
    __syncwarp();
    l.n = 0;
}

// ---------------------------------------------------------------------------
// prep_kernel: this step's stamps -> the active list.  A CTA covers
// 8 x 2048 columns: one bulk copy (TMA, cp.async.bulk) brings their 16 KB of
// stamps into shared memory on an mbarrier; warp w takes a contiguous 2048,
// in round r lane l reads the 4-byte word of columns base_w + 128 r + 4 l and
// compares its bytes with __vcmpeq4, keeping a 4-bit mask per round in one
// 64-bit register.  One atomic per CTA reserves its part of the list, the
// warps' offsets come from one shared exchange, and each warp then places
// its matches round by round with shuffle scans (no further CTA barrier),
// every round one contiguous run of the list.  Nothing downstream depends
// on the list order (the statistics are order-independent).  A full step
// only resets the target buffer's pool.

constexpr int kPrepTPB = 256;
#ifndef FT_PREP_ROUNDS
#define FT_PREP_ROUNDS 16
#endif
constexpr int kPrepRounds = FT_PREP_ROUNDS;
constexpr int kPrepCols = 4 * kPrepRounds;   // columns per thread

__global__ void __launch_bounds__(kPrepTPB) prep_kernel(const StepParams p) {
    __shared__ __align__(128) unsigned int s_tile[kPrepTPB * kPrepCols / 4];   // 16 KB of stamps
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ int s_warp[kPrepTPB / 32];
    __shared__ int s_base;
    // owned buffer columns [g_lo, g_hi); the CTA's 16 KB tile of stamps from
    // the 16-byte aligned column g_lo & ~15 (the stamp array is padded past
    // n, so the rounded-up tail stays inside it)
    const int g_lo = p.j_base, g_hi = p.j_base + p.n_v;
    const int c0 = (g_lo & ~15) + blockIdx.x * (kPrepTPB * kPrepCols);
    if (threadIdx.x == 0) mbar_init(&s_bar);
    __syncthreads();
    pdl_wait();
    Control* ctl = p.ws.ctl;
    if (p.check_done && vload(&ctl->done)) return;
    if (step_is_full(p)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->pool_next[p.out_id] = 0ULL;
        return;
    }
    if (threadIdx.x == 0) {
        const int span = min(kPrepTPB * kPrepCols, ((g_hi - c0) + 15) & ~15);
        bulk_load(s_tile, p.ws.stamp + c0, (unsigned)span, &s_bar);
    }
    const unsigned int pat = 0x01010101u * (unsigned char)vload(&ctl->seq);
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int tw = wi * (32 * kPrepCols);          // the warp's offset in the tile
    const int cw = c0 + tw;
    mbar_wait(&s_bar, 0);
    unsigned int x[kPrepRounds];
#pragma unroll
    for (int r = 0; r < kPrepRounds; ++r) x[r] = s_tile[(tw + 128 * r) / 4 + lane];   // beyond g_hi: masked below
    unsigned long long mm[(kPrepRounds + 15) / 16] = {};
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < kPrepRounds; ++r) {
        const int jw = cw + 128 * r + 4 * lane;
        const unsigned int e = __vcmpeq4(x[r], pat) & 0x01010101u;   // 0x01 per matching byte
        unsigned int m = (e * 0x01020408u) >> 24;                     // gathered into 4 bits
        const int hi = g_hi - jw, lo = g_lo - jw;                      // keep [g_lo, g_hi)
        if (hi < 4) m &= hi <= 0 ? 0u : (1u << hi) - 1u;
        if (lo > 0) m &= ~((1u << lo) - 1u);
        mm[r / 16] |= (unsigned long long)m << (4 * (r % 16));
        cnt += __popc(m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
    if (lane == 0) s_warp[wi] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
#pragma unroll
        for (int k = 0; k < kPrepTPB / 32; ++k) {
            const int c = s_warp[k];
            s_warp[k] = t;
            t += c;
        }
        s_base = t ? atomicAdd(&ctl->n_act, t) : 0;
    }
    __syncthreads();
    if (cnt == 0) return;
    int base = s_base + s_warp[wi];
    const unsigned int lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kPrepRounds; ++r) {
        const unsigned int m = (unsigned int)(mm[r / 16] >> (4 * (r % 16))) & 15u;
        const int c = __popc(m);
        // the lanes' exclusive prefix of c (0..4) from the ballots of its
        // three bits, no shuffle scan
        const unsigned int b0 = __ballot_sync(kFull, c & 1), b1 = __ballot_sync(kFull, c & 2),
                           b2 = __ballot_sync(kFull, c & 4);
        const int pos = base + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
        base += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
        const int jw = cw + 128 * r + 4 * lane - g_lo;
#pragma unroll
        for (int b = 0; b < 4; ++b)     // ascending columns, predicated stores
            if (m & (1u << b)) p.ws.act[pos + __popc(m & ((1u << b) - 1u))] = jw + b;
    }
}

// ---------------------------------------------------------------------------
// band_kernel: one lane per active column.
//
// Three dependent loads: the packed L^T row (and the column's own first
// value), the neighbours' row signatures, then -- for a column whose
// neighbourhood holds more than one row -- the neighbours' second rows and
// values.  A single-row neighbourhood (every non-empty neighbour holds one
// entry, of the column's own row, and phi > 0: a cell interior) is finished
// with the exact closed form v' = clamp(v) * (1 / (0 + clamp(v))) -- with
// finite couplings every term of the update cancels, so d = +-0 -- without
// reading the neighbours' values (they can only matter through the
// finiteness of Lt; values this library writes are finite unless a kernel
// raised the sticky nonfinite flag, which switches the check on).  A union
// of at most two rows with at most two entries per neighbour takes the
// straight-line two-row update, Lt accumulated branch-free in L order -- the
// reference's accumulator order.  Anything else goes to the wide list.

#ifndef FT_BAND_TPB
#define FT_BAND_TPB 128     // 128 threads x 8 CTAs per SM: +1.3 % at C3 over 256 x 4
#endif
constexpr int kBandTPB = FT_BAND_TPB;
constexpr int kWarpBuf = 128;    // warp-staged wide-list entries

template <typename T, bool UNIFORM, bool PACKED>
__device__ __forceinline__ void band_column(const StepParams& p, int jl, bool have, bool full, bool chk,
                                            unsigned char nxt, int lane, Acc& acc, long long* s_bm,
                                            WarpList& wl, int4 pk) {
    const int j = p.j_base + jl;
    // stage 1: the packed L^T row (prefetched by the caller); the column's
    // own signature and value
    const double phs = have ? ldv<T>(p.in.v0, j) : 0.0;
    const int sgj = have ? __ldg(&p.in.sig[j]) : FT_SIG_EMPTY;
    int q0 = 0;
    int u[kMD];
    const int n = unpack_lrow<PACKED>(p, pk, jl, j, have, u, q0);   // u[k] = -1 beyond n
    // stage 2: the neighbours' signatures
    int sg[kMD];
#pragma unroll
    for (int k = 0; k < kMD; ++k) sg[k] = (u[k] >= 0) ? __ldg(&p.in.sig[u[k]]) : FT_SIG_EMPTY;
    bool same = true, big = false, hasd = false;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        same &= (sg[k] == FT_SIG_EMPTY) || (sg[k] == sgj);
        big |= sg[k] <= -3;
        hasd |= u[k] == j;
    }
    const double invdeg = UNIFORM ? recip_deg(n) : 0.0;
    bool fast = have && hasd && p.cp.finite && sgj >= 0 && sgj < kPair && same && phs > 0.0;
    if (chk && fast) {
        // Lt(sgj, j) and the values must be finite for the closed form
        bool fin = true;
        double lam = 0.0;
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            if (k < n && sg[k] == sgj) {
                const double v = ldv<T>(p.in.v0, u[k]);
                fin &= isfinite(v);
                const double l = UNIFORM ? (u[k] == j ? -1.0 : invdeg) : ldv<T>(p.lap_val, q0 + k);
                lam = lam + v * l;
            }
        }
        fast = fin && isfinite(lam);
    }
    const bool wide = have && !fast && (!hasd || big);
    const bool gen = have && !fast && !wide;
    const int skc_old = (have && !full) ? __ldg(&p.ws.skc[jl]) : 0;

    bool changed = false, fin_here = false;
    double bm_new = 0.0, bm_old = 0.0;
    int cnt_new = 0, cnt_old = 0, sk_new = 0;

    // a cell interior at rest holds exactly 1.0, and 1.0 * (1 / (0 + 1.0))
    // == 1.0: a warp whose closed-form lanes all hold 1.0 skips the division
    __syncwarp();   // reconverge after the divergent finiteness check
    const bool ones = __all_sync(kFull, !fast || phs == 1.0);
    if (fast) {
        const double v = phs > 1.0 ? 1.0 : phs;
        const double nv = ones ? 1.0 : v * (1.0 / (0.0 + v));
        const bool keep = nv != 0.0;
        cnt_new = keep ? 1 : 0;
        cnt_old = 1;
        sk_new = 1;
        if (sgj == 0) {
            bm_old = phs;
            bm_new = keep ? nv : 0.0;
        }
        acc.md = fmax(acc.md, fabs(nv - phs));
        changed = !keep || !same_bits<T>(nv, phs);
        p.out.sig[j] = keep ? sgj : FT_SIG_EMPTY;
        ((T*)p.out.v0)[j] = (T)nv;
        fin_here = true;
    }
    bool more = false;
    if (gen) {
        // stage 3: second rows and values.  x = a neighbour's first row, ax
        // its second (-1 when absent)
        int x[kMD], ax[kMD];
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            x[k] = sg[k] >= 0 ? (sg[k] & ~kPair) : -1;
            ax[k] = sg[k] >= kPair ? __ldg(&p.in.aux[u[k]]) : -1;
        }
        const bool prj = sgj >= kPair;
        const int xj = sgj & ~kPair;
        const int axj = prj ? __ldg(&p.in.aux[j]) : -1;
        const double vj1 = prj ? ldv<T>(p.in.v1, j) : 0.0;
        unsigned int rlo = 0xffffffffu;   // -1 (absent) is the largest unsigned value
        int rhi = -1;
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            rlo = min(rlo, min((unsigned int)x[k], (unsigned int)ax[k]));
            rhi = max(rhi, max(x[k], ax[k]));
        }
        const int lo = (int)rlo;          // -1 when the neighbourhood is empty
        // a third row: a first row strictly between lo and rhi, or a second
        // row below rhi (absent entries, -1, compare as the largest unsigned)
        const unsigned span = rhi > lo ? (unsigned)(rhi - lo - 1) : 0u;
#pragma unroll
        for (int k = 0; k < kMD; ++k)
            more |= ((unsigned)(x[k] - lo - 1) < span) | ((unsigned)ax[k] < (unsigned)rhi);
        // Lt(lo, j), Lt(rhi, j) in L order (the reference's accumulator
        // order): every slot adds its coefficient times L(j, u), the
        // coefficient 0 when the slot holds no entry of that row -- adding
        // an exact zero leaves the sum bitwise unchanged (it is never -0)
        double l0 = 0.0, l1 = 0.0;
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            const double l = UNIFORM ? (u[k] == j ? -1.0 : invdeg)
                                     : ((k < n) ? ldv<T>(p.lap_val, q0 + k) : 0.0);
            const double a0 = x[k] >= 0 ? ldv<T>(p.in.v0, u[k]) : 0.0;
            const double a1 = ax[k] >= 0 ? ldv<T>(p.in.v1, u[k]) : 0.0;
            const double c0 = x[k] == lo ? a0 : 0.0;
            const double c1 = x[k] == rhi ? a0 : (ax[k] == rhi ? a1 : 0.0);
            l0 = l0 + c0 * l;
            l1 = l1 + c1 * l;
        }
        if (!more) {
            const int r0 = lo < 0 ? INT_MAX : lo;   // empty neighbourhood: empty skeleton
            const double p0 = (sgj >= 0 && xj == lo) ? phs : 0.0;
            const double p1 = (sgj >= 0 && xj == rhi) ? phs : ((prj && axj == rhi) ? vj1 : 0.0);
            VRes res;
            vres_init(res);
            double nv0, nv1;
            unsigned int om;
            process_two(rhi == lo ? 1 : 2, r0, rhi, p0, l0, p1, l1, p.cp, c_recip, res, nv0, nv1, om);
            report_flags(res, j, p);
            cnt_new = res.cnt;
            sk_new = res.nskel;
            bm_new = res.bm;
            acc.md = fmax(acc.md, res.maxd);
            int ns = FT_SIG_EMPTY, na = 0;
            double y0 = 0.0, y1 = 0.0;
            if (om == 3u) { ns = lo | kPair; na = rhi; y0 = nv0; y1 = nv1; }
            else if (om == 1u) { ns = lo; y0 = nv0; }
            else if (om == 2u) { ns = rhi; y0 = nv1; }
            cnt_old = sig_count(sgj);
            bm_old = (sgj >= 0 && xj == 0) ? phs : 0.0;
            changed = ns != sgj || (cnt_new >= 1 && !same_bits<T>(y0, phs)) ||
                      (cnt_new == 2 && (na != axj || !same_bits<T>(y1, vj1)));
            p.out.sig[j] = ns;
            if (cnt_new >= 1) ((T*)p.out.v0)[j] = (T)y0;
            if (cnt_new == 2) { p.out.aux[j] = na; ((T*)p.out.v1)[j] = (T)y1; }
            if (!isfinite(y0) || !isfinite(y1)) atomicOr(&p.ws.ctl->nonfinite, 1u);
            fin_here = true;
        }
    }
    __syncwarp();   // reconverge after the per-lane paths before the collectives
    wlist_push(wide || (gen && more), j, wl, lane);
    if (fin_here) {
        acc.dn += cnt_new - (full ? 0 : cnt_old);
        acc.ds += sk_new - (full ? 0 : skc_old);
        if (p.track && (full || sk_new != skc_old)) p.ws.skc[jl] = sk_new;
        if (p.track && changed) mark_ring(p, u, n, nxt);
    }
    bm_fold(fin_here ? bm_new : 0.0, fin_here ? bm_old : 0.0, full, s_bm);
}

#ifndef FT_BAND_MINB
#define FT_BAND_MINB (1024 / FT_BAND_TPB)   // 64 registers: 1024 threads per SM
#endif
template <typename T, bool UNIFORM, bool PACKED, int MINB = FT_BAND_MINB>
__global__ void __launch_bounds__(kBandTPB, MINB) band_kernel(const StepParams p) {
    pdl_wait();
    Control* ctl = p.ws.ctl;
    __shared__ long long s_bm[4];
    __shared__ double s_md[kBandTPB / 32];
    __shared__ long long s_cnt[2 * (kBandTPB / 32)];
    __shared__ int s_wl[kBandTPB / 32][kWarpBuf];
    if (p.check_done && vload(&ctl->done)) return;
    if (threadIdx.x < 4) s_bm[threadIdx.x] = 0;
    __syncthreads();
    WarpList wl{s_wl[threadIdx.x >> 5], 0};
    const bool full = step_is_full(p);
    const int n_act = full ? p.n_v : vload(&ctl->n_act);
    const bool chk = p.force_check || vload(&ctl->nonfinite);
    const unsigned char nxt = (unsigned char)(vload(&ctl->seq) + 1);
    const int lane = threadIdx.x & 31;
    Acc acc;
    acc_init(acc);
    // chunks of kBandTPB columns; the next chunk's column index and packed L
    // row are loaded before the current chunk is processed, taking two
    // levels off its load chain
    const int stride = gridDim.x * kBandTPB;
    int c = blockIdx.x * kBandTPB;
    bool have = c + (int)threadIdx.x < n_act;
    int jl = have ? (full ? c + (int)threadIdx.x : __ldg(&p.ws.act[c + threadIdx.x])) : 0;
    int4 pk = make_int4(0, 0, 0, 0);
    if (PACKED && have) pk = __ldg(&p.lap_pack[jl]);
    for (; c < n_act; c += stride) {
        const int in = c + stride + (int)threadIdx.x;
        const bool hn = in < n_act;
        const int jn = hn ? (full ? in : __ldg(&p.ws.act[in])) : 0;
        int4 pn = make_int4(0, 0, 0, 0);
        if (PACKED && hn) pn = __ldg(&p.lap_pack[jn]);
        band_column<T, UNIFORM, PACKED>(p, jl, have, full, chk, nxt, lane, acc, s_bm, wl, pk);
        if (wl.n > kWarpBuf - 32) wlist_flush(wl, &ctl->n_wide, p.ws.wide, lane);
        have = hn;
        jl = jn;
        pk = pn;
    }
    wlist_flush(wl, &ctl->n_wide, p.ws.wide, lane);
    __syncthreads();
    acc_flush<kBandTPB>(acc, s_bm, s_md, s_cnt, ctl);
}

// ---------------------------------------------------------------------------
// pool placement of a column with cnt > 2 entries: an active step reuses the
// column's own range in the target buffer (its value of two steps ago) when
// it is large enough; otherwise fresh entries.  Returns -1 on overflow.

__device__ __forceinline__ long long pool_take(const StepParams& p, int j, int cnt, bool full) {
    if (!full) {
        const int os = p.out.sig[j];
        if (os <= -cnt) return (long long)p.out.aux[j];
    }
    const long long off = (long long)atomicAdd(&p.ws.ctl->pool_next[p.out_id], (unsigned long long)cnt);
    if (off + cnt > p.cap) {
        atomicExch(&p.ws.ctl->overflow, 1);
        return -1;
    }
    return off;
}

// the same for one column per lane (cnt <= 2: none), fresh entries taken
// with one atomic per warp (warp-collective)
__device__ __forceinline__ long long pool_take_warp(const StepParams& p, int j, int cnt, bool full, int lane) {
    long long off = -1;
    int need = cnt > 2 ? cnt : 0;
    if (need && !full) {
        const int os = p.out.sig[j];
        if (os <= -cnt) { off = (long long)p.out.aux[j]; need = 0; }
    }
    int incl = need;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    const int tot = __shfl_sync(kFull, incl, 31);
    if (tot == 0) return off;
    long long base = 0;
    if (lane == 31) base = (long long)atomicAdd(&p.ws.ctl->pool_next[p.out_id], (unsigned long long)tot);
    base = __shfl_sync(kFull, base, 31);
    if (base + tot > p.cap) {
        if (lane == 31) atomicExch(&p.ws.ctl->overflow, 1);
        return need ? -1 : off;
    }
    return need ? base + incl - need : off;
}

// ---------------------------------------------------------------------------
// wide3_kernel: the band kernel's listed columns, one lane per column: at
// most three rows in the union and at most three entries per neighbour
// (a neighbour with three entries is read from the pool).  Lt of the rows
// rlo < rmid < rhi accumulated in L order, then the generic window update
// (process_window<3>).  Anything wider goes on to the warp kernel.

template <typename T, bool UNIFORM, bool PACKED, bool OWN>
__device__ __forceinline__ void wide3_column(const StepParams& p, int j, bool have, bool full, unsigned char nxt,
                                             int lane, Acc& acc, long long* s_bm, int4 pk) {
    const int jl = j - p.j_base;
    int q0 = 0;
    int u[kMD];
    const int n = unpack_lrow<PACKED>(p, pk, jl, j, have, u, q0);
    int sg[kMD], ax[kMD];
#pragma unroll
    for (int k = 0; k < kMD; ++k) sg[k] = (k < n) ? __ldg(&p.in.sig[u[k]]) : FT_SIG_EMPTY;
#pragma unroll
    for (int k = 0; k < kMD; ++k) ax[k] = (sg[k] >= kPair || sg[k] <= -3) ? __ldg(&p.in.aux[u[k]]) : 0;
    int kd = -1;
    bool ok = have && n > 0;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        kd = (k < n && u[k] == j) ? k : kd;
        ok &= sg[k] >= -3;
    }
    ok &= kd >= 0;
    // the rows of every neighbour (ascending), INT_MAX when absent
    int rr[kMD][3];
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        const int s = ok ? sg[k] : FT_SIG_EMPTY;
        rr[k][0] = s >= 0 ? (s & ~kPair) : (s == -3 ? __ldg(&p.in.pidx[ax[k]]) : INT_MAX);
        rr[k][1] = s >= kPair ? ax[k] : (s == -3 ? __ldg(&p.in.pidx[ax[k] + 1]) : INT_MAX);
        rr[k][2] = s == -3 ? __ldg(&p.in.pidx[ax[k] + 2]) : INT_MAX;
    }
    // rlo / rhi over the present rows (absent = INT_MAX), then the rows
    // strictly between them: their minimum is the middle row, a larger one
    // means a fourth row (branch-free min / max chains)
    int rlo = INT_MAX, rhi = -1;
#pragma unroll
    for (int k = 0; k < kMD; ++k)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int r = rr[k][t];
            rlo = min(rlo, r);
            rhi = max(rhi, r != INT_MAX ? r : -1);
        }
    int rmid = INT_MAX, rmax_mid = -1;
#pragma unroll
    for (int k = 0; k < kMD; ++k)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int r = rr[k][t];
            const bool mid = r > rlo && r < rhi;
            rmid = min(rmid, mid ? r : INT_MAX);
            rmax_mid = max(rmax_mid, mid ? r : -1);
        }
    const bool more = rmax_mid > rmid && rmid != INT_MAX;
    const bool run = ok && !more;
    // Lt per row in L order; PHI(r, j) and the old entries through u == j
    const double invdeg = UNIFORM ? recip_deg(n) : 0.0;
    double l0 = 0.0, l1 = 0.0, l2 = 0.0, p0 = 0.0, p1 = 0.0, p2 = 0.0;
    int sgj = FT_SIG_EMPTY, axj = 0;
    double oj[3] = {0.0, 0.0, 0.0};
    int orr[3] = {INT_MAX, INT_MAX, INT_MAX};
    if (run) {
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            if (k >= n) continue;
            const double l = lap_value<T, UNIFORM>(p, k, kd, q0, invdeg);
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int r = rr[k][t];
                if (r == INT_MAX) continue;
                const double a = hyb_val<T>(p.in, u[k], sg[k], ax[k], t);
                if (OWN) {
                    if (r == rlo) l0 = l0 + a * l;
                    else if (r == rhi) l2 = l2 + a * l;
                    else l1 = l1 + a * l;
                } else {
                    if (k == kd) { oj[t] = a; orr[t] = r; }
                    if (r == rlo) { l0 = l0 + a * l; if (k == kd) p0 = a; }
                    else if (r == rhi) { l2 = l2 + a * l; if (k == kd) p2 = a; }
                    else { l1 = l1 + a * l; if (k == kd) p1 = a; }
                }
            }
            if (!OWN && k == kd) { sgj = sg[k]; axj = ax[k]; }
        }
        if (OWN) {
        // the column's own entries (<= 3, rows ascending, a subset of
        // rlo / rmid / rhi), re-read (L1) instead of tracked through the
        // neighbour loop: PHI(r, j) per window row.  Fewer registers (117
        // against 128), which the dense-band variant's fifth CTA per SM needs
        sgj = __ldg(&p.in.sig[j]);
        axj = (sgj >= kPair || sgj <= -3) ? __ldg(&p.in.aux[j]) : 0;
        const int cj = sig_count(sgj);
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if (t < cj) { orr[t] = hyb_row<T>(p.in, sgj, axj, t); oj[t] = hyb_val<T>(p.in, j, sgj, axj, t); }
        p0 = orr[0] == rlo ? oj[0] : 0.0;
        p1 = rmid == INT_MAX ? 0.0 : (orr[0] == rmid ? oj[0] : (orr[1] == rmid ? oj[1] : 0.0));
        p2 = orr[0] == rhi ? oj[0] : (orr[1] == rhi ? oj[1] : (orr[2] == rhi ? oj[2] : 0.0));
        }
    }
    Win<3> w;
    w.more = false;
    if (rlo == INT_MAX) {
        w.m = 0;
    } else if (rlo == rhi) {
        w.m = 1;
        w.rows[0] = rlo; w.lam[0] = l0; w.phi[0] = p0;
    } else if (rmid == INT_MAX) {
        w.m = 2;
        w.rows[0] = rlo; w.lam[0] = l0; w.phi[0] = p0;
        w.rows[1] = rhi; w.lam[1] = l2; w.phi[1] = p2;
    } else {
        w.m = 3;
        w.rows[0] = rlo; w.lam[0] = l0; w.phi[0] = p0;
        w.rows[1] = rmid; w.lam[1] = l1; w.phi[1] = p1;
        w.rows[2] = rhi; w.lam[2] = l2; w.phi[2] = p2;
    }
    VRes res;
    vres_init(res);
    unsigned int om = 0;
    if (run) {
        process_window<3>(w, p.cp, res, om, c_recip);
        report_flags(res, j, p);
    }
    __syncwarp();
    list_push(have && !run, j, &p.ws.ctl->n_w2, p.ws.w2, lane);
    const int cnt = __popc(om);
    const long long off = pool_take_warp(p, j, run ? cnt : 0, full, lane);
    // the new entries in row order; the change test against the old ones
    int nr[3] = {0, 0, 0};
    double nv[3] = {0.0, 0.0, 0.0};
    {
        int q = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (om & (1u << i)) {
                if (q == 0) { nr[0] = w.rows[i]; nv[0] = w.lam[i]; }
                else if (q == 1) { nr[1] = w.rows[i]; nv[1] = w.lam[i]; }
                else { nr[2] = w.rows[i]; nv[2] = w.lam[i]; }
                ++q;
            }
        }
    }
    const int co = sig_count(sgj);
    bool changed = run && cnt != co;
#pragma unroll
    for (int i = 0; i < 3; ++i)
        if (run && i < cnt && i < co) changed |= nr[i] != orr[i] || !same_bits<T>(nv[i], oj[i]);
    double bm_new = 0.0, bm_old = 0.0;
    if (run) {
        bm_new = res.bm;
        bm_old = (co > 0 && orr[0] == 0) ? oj[0] : 0.0;
        acc.md = fmax(acc.md, res.maxd);
        const int skc_old = full ? 0 : p.ws.skc[jl];
        acc.dn += cnt - (full ? 0 : co);
        acc.ds += res.nskel - skc_old;
        if (p.track && (full || res.nskel != skc_old)) p.ws.skc[jl] = res.nskel;
        if (p.track && changed) mark_ring(p, u, n, nxt);
        bool nf = false;
        if (cnt <= 2) {
            p.out.sig[j] = cnt == 0 ? FT_SIG_EMPTY : (cnt == 2 ? (nr[0] | kPair) : nr[0]);
            if (cnt >= 1) ((T*)p.out.v0)[j] = (T)nv[0];
            if (cnt == 2) { p.out.aux[j] = nr[1]; ((T*)p.out.v1)[j] = (T)nv[1]; }
            nf = !isfinite(nv[0]) || !isfinite(nv[1]);
        } else if (off >= 0) {
            p.out.sig[j] = -3;
            p.out.aux[j] = (int)off;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                p.out.pidx[off + i] = nr[i];
                ((T*)p.out.pval)[off + i] = (T)nv[i];
                nf |= !isfinite(nv[i]);
            }
        }
        if (nf) atomicOr(&p.ws.ctl->nonfinite, 1u);
    }
    __syncwarp();
    bm_fold(bm_new, bm_old, full, s_bm);
}

#ifndef FT_W3_TPB
#define FT_W3_TPB 128
#endif
constexpr int kWide3TPB = FT_W3_TPB;
#ifndef FT_W3_MINB
#define FT_W3_MINB (512 / FT_W3_TPB)
#endif

// FT_HINT_DENSE_BAND: 5 CTAs per SM (96 registers, a few spills) and the
// own-entry re-read -- +4 % at C5 (1.7M listed columns, ~18 passes of the
// grid), -0.7 % at C3 (190K, ~2 passes), so it is chosen by the hint
constexpr int kWide3DenseMinB = 640 / FT_W3_TPB;

template <typename T, bool UNIFORM, bool PACKED, bool OWN>
__device__ __forceinline__ void wide3_body(const StepParams& p) {
    pdl_wait();
    Control* ctl = p.ws.ctl;
    __shared__ long long s_bm[4];
    __shared__ double s_md[kWide3TPB / 32];
    __shared__ long long s_cnt[2 * (kWide3TPB / 32)];
    if (p.check_done && vload(&ctl->done)) return;
    const int nc = vload(&ctl->n_wide);
    if ((int)blockIdx.x * kWide3TPB >= nc) return;
    if (threadIdx.x < 4) s_bm[threadIdx.x] = 0;
    __syncthreads();
    const bool full = step_is_full(p);
    const unsigned char nxt = (unsigned char)(vload(&ctl->seq) + 1);
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * kWide3TPB;
    Acc acc;
    acc_init(acc);
    // the next column's index and packed L row are loaded before the current
    // column is processed (two levels off its load chain, as in the band kernel)
    int i = blockIdx.x * kWide3TPB + threadIdx.x;
    bool have = i < nc;
    int j = have ? __ldg(&p.ws.wide[i]) : p.j_base;
    int4 pk = make_int4(0, 0, 0, 0);
    if (PACKED && have) pk = __ldg(&p.lap_pack[j - p.j_base]);
    for (int i0 = blockIdx.x * kWide3TPB; i0 < nc; i0 += stride) {
        const int in = i + stride;
        const bool hn = in < nc;
        const int jn = hn ? __ldg(&p.ws.wide[in]) : p.j_base;
        int4 pn = make_int4(0, 0, 0, 0);
        if (PACKED && hn) pn = __ldg(&p.lap_pack[jn - p.j_base]);
        wide3_column<T, UNIFORM, PACKED, OWN>(p, j, have, full, nxt, lane, acc, s_bm, pk);
        i = in;
        have = hn;
        j = jn;
        pk = pn;
    }
    __syncthreads();
    acc_flush<kWide3TPB>(acc, s_bm, s_md, s_cnt, ctl);
}

template <typename T, bool UNIFORM, bool PACKED>
__global__ void __launch_bounds__(kWide3TPB, FT_W3_MINB) wide3_kernel(const StepParams p) {
    wide3_body<T, UNIFORM, PACKED, false>(p);
}

template <typename T, bool UNIFORM, bool PACKED>
__global__ void __launch_bounds__(kWide3TPB, kWide3DenseMinB) wide3_dense_kernel(const StepParams p) {
    wide3_body<T, UNIFORM, PACKED, true>(p);
}

// ---------------------------------------------------------------------------
// wide4_kernel: the three-row kernel's leftovers, one lane per column: at
// most four rows in the union and four entries per neighbour (the C5 band's
// junction columns).  (The same generic window at K = 3 in place of the
// three-row kernel is 5-16 % slower: its min / mid / max form stays.)  The neighbourhood goes through the sorted register
// window (win_insert, L order: each row's Lt in the reference's order) and
// process_window<4>; anything wider goes on to the warp kernel (the wide[]
// list, consumed by then).

#ifndef FT_W4_TPB
#define FT_W4_TPB 128
#endif
constexpr int kWide4TPB = FT_W4_TPB;
// below this many leftovers of the three-row kernel the warp kernel takes
// them all directly (few columns: one warp each finishes sooner than a
// latency-bound lane-per-column pass followed by the warp kernel)
constexpr int kWide4Min = 49152;

template <typename T, bool UNIFORM, bool PACKED, int K>
__device__ __forceinline__ void widek_column(const StepParams& p, int j, bool have, bool full, unsigned char nxt,
                                             int lane, Acc& acc, long long* s_bm, int* out_count, int* out_list) {
    const int jl = j - p.j_base;
    int4 pk = make_int4(0, 0, 0, 0);
    if (PACKED && have) pk = __ldg(&p.lap_pack[jl]);
    int q0 = 0;
    int u[kMD];
    const int n = unpack_lrow<PACKED>(p, pk, jl, j, have, u, q0);
    int sg[kMD], ax[kMD];
#pragma unroll
    for (int k = 0; k < kMD; ++k) sg[k] = (k < n) ? __ldg(&p.in.sig[u[k]]) : FT_SIG_EMPTY;
#pragma unroll
    for (int k = 0; k < kMD; ++k) ax[k] = (sg[k] >= kPair || sg[k] < -1) ? __ldg(&p.in.aux[u[k]]) : 0;
    int kd = -1;
    bool ok = have && n > 0;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        kd = (k < n && u[k] == j) ? k : kd;
        ok &= sg[k] >= -K;
    }
    ok &= kd >= 0;
    const double invdeg = UNIFORM ? recip_deg(n) : 0.0;
    Win<K> w;
    w.m = 0;
    w.more = false;
    if (ok) {
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            if (k >= n) continue;
            const double l = lap_value<T, UNIFORM>(p, k, kd, q0, invdeg);
            const int c = sig_count(sg[k]);
            for (int t = 0; t < c; ++t) {
                const double a = hyb_val<T>(p.in, u[k], sg[k], ax[k], t);
                win_insert<K>(w, hyb_row<T>(p.in, sg[k], ax[k], t), a * l, k == kd, a);
            }
        }
    }
    const bool run = ok && !w.more;
    VRes res;
    vres_init(res);
    unsigned int om = 0;
    if (run) {
        process_window<K>(w, p.cp, res, om, c_recip);
        report_flags(res, j, p);
    }
    __syncwarp();
    list_push(have && !run, j, out_count, out_list, lane);
    const int cnt = __popc(om);
    const long long off = pool_take_warp(p, j, run ? cnt : 0, full, lane);
    // the column's old entries (through u == j) for the change test
    int sgj = FT_SIG_EMPTY, axj = 0;
#pragma unroll
    for (int k = 0; k < kMD; ++k)
        if (k == kd) { sgj = sg[k]; axj = ax[k]; }
    const int co = sig_count(sgj);
    bool changed = run && cnt != co;
    double bm_new = 0.0, bm_old = 0.0;
    if (run) {
        bool nf = false;
        int q = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (!(om & (1u << i))) continue;
            const int r = w.rows[i];
            const double nv = w.lam[i];
            if (q < co) changed |= hyb_row<T>(p.in, sgj, axj, q) != r ||
                                   !same_bits<T>(nv, hyb_val<T>(p.in, j, sgj, axj, q));
            nf |= !isfinite(nv);
            if (cnt <= 2) {
                if (q == 0) {
                    p.out.sig[j] = cnt == 2 ? (r | kPair) : r;
                    ((T*)p.out.v0)[j] = (T)nv;
                } else {
                    p.out.aux[j] = r;
                    ((T*)p.out.v1)[j] = (T)nv;
                }
            } else if (off >= 0) {
                p.out.pidx[off + q] = r;
                ((T*)p.out.pval)[off + q] = (T)nv;
            }
            ++q;
        }
        if (cnt == 0) p.out.sig[j] = FT_SIG_EMPTY;
        else if (cnt > 2 && off >= 0) { p.out.sig[j] = -cnt; p.out.aux[j] = (int)off; }
        if (nf) atomicOr(&p.ws.ctl->nonfinite, 1u);
        bm_new = res.bm;
        bm_old = (co > 0 && hyb_row<T>(p.in, sgj, axj, 0) == 0) ? hyb_val<T>(p.in, j, sgj, axj, 0) : 0.0;
        acc.md = fmax(acc.md, res.maxd);
        const int skc_old = full ? 0 : p.ws.skc[jl];
        acc.dn += cnt - (full ? 0 : co);
        acc.ds += res.nskel - skc_old;
        if (p.track && (full || res.nskel != skc_old)) p.ws.skc[jl] = res.nskel;
        if (p.track && changed) mark_ring(p, u, n, nxt);
    }
    __syncwarp();
    bm_fold(bm_new, bm_old, full, s_bm);
}

template <typename T, bool UNIFORM, bool PACKED>
#ifndef FT_W4_MINB
#define FT_W4_MINB (768 / FT_W4_TPB)      // 80 registers: 768 threads per SM (+1.6 % at C5 over 512)
#endif
__global__ void __launch_bounds__(kWide4TPB, FT_W4_MINB) wide4_kernel(const StepParams p) {
    pdl_wait();
    Control* ctl = p.ws.ctl;
    __shared__ long long s_bm[4];
    __shared__ double s_md[kWide4TPB / 32];
    __shared__ long long s_cnt[2 * (kWide4TPB / 32)];
    if (p.check_done && vload(&ctl->done)) return;
    const int nc = vload(&ctl->n_w2);
    if (nc < p.wide4_min || (int)blockIdx.x * kWide4TPB >= nc) return;
    if (threadIdx.x < 4) s_bm[threadIdx.x] = 0;
    __syncthreads();
    const bool full = step_is_full(p);
    const unsigned char nxt = (unsigned char)(vload(&ctl->seq) + 1);
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * kWide4TPB;
    Acc acc;
    acc_init(acc);
    for (int i0 = blockIdx.x * kWide4TPB; i0 < nc; i0 += stride) {
        const int i = i0 + threadIdx.x;
        const bool have = i < nc;
        widek_column<T, UNIFORM, PACKED, 4>(p, have ? __ldg(&p.ws.w2[i]) : p.j_base, have, full, nxt, lane, acc,
                                            s_bm, &ctl->n_w3, p.ws.wide);
    }
    __syncthreads();
    acc_flush<kWide4TPB>(acc, s_bm, s_md, s_cnt, ctl);
}

// ---------------------------------------------------------------------------
// the exact windowed algorithm (no width limit) for the rare column whose
// neighbourhood exceeds the wide kernel's staging capacity: ascending row
// windows of K rows gathered from global memory, aggregates first, then the
// update and the normaliser, then the emit pass.

// a column's neighbourhood entries from the CSR and the hybrid field
template <typename T, bool UNIFORM>
struct GlobalSrc {
    const StepParams& p;
    int j;
    // rows r > lo of the union of PHI(:, u), u in L^T(:, j), with the Lt
    // accumulation, into the window (the K smallest such rows)
    template <int K>
    __device__ __forceinline__ void gather(Win<K>& w, int lo) const {
        w.m = 0;
        w.more = false;
        const int q0 = __ldg(&p.lap_ptr[j - p.j_base]);   // L rows are local to the domain
        const int q1 = __ldg(&p.lap_ptr[j - p.j_base + 1]);
        const double invdeg = UNIFORM ? 1.0 / (double)(q1 - q0 - 1) : 0.0;
        for (int q = q0; q < q1; ++q) {
            const int u = __ldg(&p.lap_idx[q]);
            const bool diag = (u == j);
            double l;
            if (UNIFORM) l = diag ? -1.0 : invdeg;
            else l = ldv<T>(p.lap_val, q);
            const int s = __ldg(&p.in.sig[u]);
            const int cnt = sig_count(s);
            const int a = cnt >= 2 ? __ldg(&p.in.aux[u]) : 0;
            for (int c = 0; c < cnt; ++c) {
                const int r = hyb_row<T>(p.in, s, a, c);
                if (r <= lo) continue;
                const double ph = hyb_val<T>(p.in, u, s, a, c);
                win_insert<K>(w, r, ph * l, diag, ph);
            }
        }
    }
};

// One column through the windowed algorithm.  emit == false: statistics
// only (res.cnt = output entries); emit == true: writes column j (the pool
// range at poff when res.cnt > 2).  `changed`: the result differs from the
// column's input entries.
template <typename T, int K, class Src>
__device__ __noinline__ void vertex_slow(int j, const StepParams& p, const Src& src, VRes& res, long long poff,
                                         bool emit, bool& changed) {
    Win<K> w;
    Agg g;
    agg_init(g);
    int lo = -1;
    do {
        src.gather(w, lo);
        pass_aggregate<K>(w, g);
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    const int cnt_known = res.cnt;
    res.nskel = g.n;
    res.bad_phi_row = g.bad_phi_row;
    res.bad_lt_row = g.bad_lt_row;
    res.nan = false;
    res.cnt = 0; res.bm = 0.0; res.maxd = 0.0;
    // the column's old entries, for the change test
    const int so = __ldg(&p.in.sig[j]);
    const int co = sig_count(so);
    const int ao = co >= 2 ? __ldg(&p.in.aux[j]) : 0;
    changed = false;
    int r0 = 0, r1 = 0;
    double x0 = 0.0, x1 = 0.0;
    if (g.n == 0) {
        changed = co != 0;
        if (emit) p.out.sig[j] = FT_SIG_EMPTY;
        return;
    }
    const Coef c = make_coef(g, p.cp, nullptr);
    double s = 0.0;
    lo = -1;
    do {
        src.gather(w, lo);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            s = s + update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p.cp, res.nan);
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    const bool spos = s > 0.0;
    const double inv = recip_pos(spos, s);
    bool dummy = false;
    lo = -1;
    do {
        src.gather(w, lo);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            const double v = update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p.cp, dummy);
            const double nv = spos ? v * inv : v;
            if (nv != 0.0) {
                const int k = res.cnt;
                if (k >= co || hyb_row<T>(p.in, so, ao, k) != w.rows[i] ||
                    !same_bits<T>(nv, hyb_val<T>(p.in, j, so, ao, k)))
                    changed = true;
                if (emit) {
                    if (cnt_known <= 2) {
                        if (k == 0) { r0 = w.rows[i]; x0 = nv; }
                        else { r1 = w.rows[i]; x1 = nv; }
                    } else {
                        p.out.pidx[poff + k] = w.rows[i];
                        ((T*)p.out.pval)[poff + k] = (T)nv;
                        if (!isfinite(nv)) atomicOr(&p.ws.ctl->nonfinite, 1u);
                    }
                }
                res.cnt++;
                if (w.rows[i] == 0) res.bm = res.bm + nv;
            }
            const double dd = fabs(nv - ph);
            if (dd > res.maxd) res.maxd = dd;
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    if (res.cnt != co) changed = true;
    if (emit) {
        if (res.cnt == 0) {
            p.out.sig[j] = FT_SIG_EMPTY;
        } else if (res.cnt <= 2) {
            p.out.sig[j] = res.cnt == 2 ? (r0 | kPair) : r0;
            ((T*)p.out.v0)[j] = (T)x0;
            if (res.cnt == 2) { p.out.aux[j] = r1; ((T*)p.out.v1)[j] = (T)x1; }
            if (!isfinite(x0) || !isfinite(x1)) atomicOr(&p.ws.ctl->nonfinite, 1u);
        } else {
            p.out.sig[j] = -res.cnt;
            p.out.aux[j] = (int)poff;
        }
    }
}

// base mass of column j of the input (its row-0 entry)
template <typename T>
__device__ __forceinline__ double base_of(const HybIn& h, int j) {
    const int s = __ldg(&h.sig[j]);
    const int c = sig_count(s);
    if (c == 0) return 0.0;
    const int a = c >= 2 ? __ldg(&h.aux[j]) : 0;
    return hyb_row<T>(h, s, a, 0) == 0 ? hyb_val<T>(h, j, s, a, 0) : 0.0;
}

// ---------------------------------------------------------------------------
// wide_kernel: the columns the three-row kernel hands on (more than three
// rows in the union, or a neighbour with more than three entries), one warp
// per column.  The warp stages the neighbourhood in shared memory -- every
// entry of every u in L^T(:, j) in L order (rows ascending within a
// neighbour) with its product PHI(r, u) L(j, u) -- then ranks the entries by
// (row, staging order): entries of one row are then consecutive and in L
// order, so each row's Lt is a sequential sum in the reference's order
// (_kernels.py:36-50).  The column aggregates and the normaliser are
// sequential sums over the rows in ascending order (_kernels.py:179-282),
// computed redundantly by every lane from shared memory; the per-row update
// is lane-parallel.  A neighbourhood beyond the staging capacity runs the
// exact windowed algorithm (vertex_slow) from global memory on lane 0.

#ifndef FT_WIDE_TPB
#define FT_WIDE_TPB 128
#endif
constexpr int kWideTPB = FT_WIDE_TPB;
constexpr int kWideWarps = kWideTPB / 32;
constexpr int kStageCap = 128;    // staged neighbourhood entries per warp

// row/ph are dead once the per-row slots are built (after a __syncwarp),
// so rpos/rv reuse them: 5.5 KB per warp, eight 4-warp CTAs per SM fit
struct WideStage {
    union {
        int row[kStageCap];       // staged entries' rows
        int rpos[kStageCap];      // output position of the row (-1: dropped)
    };
    double prod[kStageCap];       // PHI(r, u) * L(j, u)
    union {
        double ph[kStageCap];     // PHI(r, u) when u == j
        double rv[kStageCap];     // the row's new value
    };
    unsigned char diag[kStageCap];
    short order[kStageCap];       // staged index of the k-th entry in (row, L order)
    int rrow[kStageCap];          // per distinct row, ascending
    double rlam[kStageCap], rphi[kStageCap];
};

// exclusive warp scan of v with a running carry
__device__ __forceinline__ int warp_excl_scan(int v, int lane, int& total) {
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    total = __shfl_sync(kFull, incl, 31);
    return incl - v;
}

// the statistics, pool placement, emit and marks of a column beyond the
// staging capacity (lane 0, global memory)
template <typename T, bool UNIFORM>
__device__ __forceinline__ void deep_column(const StepParams& p, int j, bool full, unsigned char nxt, Acc& acc,
                                            double& bm_new, double& bm_old) {
    const int jl = j - p.j_base;
    const GlobalSrc<T, UNIFORM> src{p, j};
    VRes res;
    vres_init(res);
    bool changed = false;
    vertex_slow<T, 8>(j, p, src, res, 0, false, changed);
    report_flags(res, j, p);
    bm_new = res.bm;
    bm_old = base_of<T>(p.in, j);
    const int co = sig_count(__ldg(&p.in.sig[j]));
    const int skc_old = full ? 0 : p.ws.skc[jl];
    acc.md = fmax(acc.md, res.maxd);
    acc.dn += res.cnt - (full ? 0 : co);
    acc.ds += res.nskel - skc_old;
    if (p.track && (full || res.nskel != skc_old)) p.ws.skc[jl] = res.nskel;
    long long off = 0;
    if (res.cnt > 2) off = pool_take(p, j, res.cnt, full);
    if (off >= 0) {
        VRes r2 = res;
        bool ch2;
        vertex_slow<T, 8>(j, p, src, r2, off, true, ch2);
    }
    if (p.track && changed) {
        const int q0 = __ldg(&p.lap_ptr[jl]), q1 = __ldg(&p.lap_ptr[jl + 1]);
        for (int q = q0; q < q1; ++q) p.ws.stamp[__ldg(&p.lap_idx[q])] = nxt;
    }
}

template <typename T, bool UNIFORM, bool PACKED>
__device__ __forceinline__ void staged_column(const StepParams& p, int j, WideStage& st, bool full,
                                              unsigned char nxt, int lane, Acc& acc, long long* s_bm) {
    const int jl = j - p.j_base;
    // lane 0's bookkeeping loads, issued now so they overlap the staging:
    // the column's last skeleton size and its slot in the target buffer
    // (pool range reuse)
    int skc_pre = 0, osig = 0, oaux = 0;
    if (lane == 0) {
        skc_pre = full ? 0 : p.ws.skc[jl];
        osig = p.out.sig[j];
        oaux = p.out.aux[j];
    }
    // the L^T column: the packed row (lanes 0..7) or the CSR
    int n = 0, q0 = 0, pu = -1;
    if (PACKED) {
        const int4 pk = __ldg(&p.lap_pack[jl]);
        const int w = (lane >> 1) == 0 ? pk.x : ((lane >> 1) == 1 ? pk.y : ((lane >> 1) == 2 ? pk.z : pk.w));
        const int d = (lane & 1) ? (w >> 16) : ((int)(w << 16) >> 16);
        const bool valid = lane < kMD && d != kPackEmpty;
        pu = valid ? j + d : -1;
        n = __popc(__ballot_sync(kFull, valid));           // valid slots lead
    }
    if (n == 0) {
        q0 = __ldg(&p.lap_ptr[jl]);
        n = __ldg(&p.lap_ptr[jl + 1]) - q0;
        pu = -1;
    }
    const double invdeg = UNIFORM ? 1.0 / (double)(n - 1) : 0.0;
    // 1. stage, 32 L entries at a time
    int E = 0;
    for (int kc = 0; kc < n; kc += 32) {
        const int k = kc + lane;
        int u = 0, sgu = FT_SIG_EMPTY, au = 0, cu = 0;
        if (k < n) {
            u = pu >= 0 ? pu : __ldg(&p.lap_idx[q0 + k]);
            sgu = __ldg(&p.in.sig[u]);
            cu = sig_count(sgu);
            au = cu >= 2 ? __ldg(&p.in.aux[u]) : 0;
        }
        int tot;
        const int e0 = E + warp_excl_scan(cu, lane, tot);
        if (k < n && e0 + cu <= kStageCap) {
            const double l = UNIFORM ? (u == j ? -1.0 : invdeg) : ldv<T>(p.lap_val, q0 + k);
            for (int t = 0; t < cu; ++t) {
                const double v = hyb_val<T>(p.in, u, sgu, au, t);
                st.row[e0 + t] = hyb_row<T>(p.in, sgu, au, t);
                st.prod[e0 + t] = v * l;
                st.ph[e0 + t] = v;
                st.diag[e0 + t] = u == j;
            }
        }
        E += tot;
    }
    __syncwarp();
    if (E > kStageCap) {           // the deep kernel takes it (its list reuses act)
        if (lane == 0) p.ws.act[atomicAdd(&p.ws.ctl->n_deep, 1)] = j;
        return;
    }
    Agg g;
    agg_init(g);
    int M = 0, cnt = 0;
    double md = 0.0, bm_new = 0.0;
    bool changed = false, anynan = false;
    const int so = __ldg(&p.in.sig[j]);
    const int co = sig_count(so);
    const int ao = co >= 2 ? __ldg(&p.in.aux[j]) : 0;
    if (E <= 32) {
        // 2-5 with one staged entry per lane: rows grouped by __match_any_sync
        // (a row's entries are its group's lanes in staging = L order), one
        // lane per distinct row, the row-order sums by shuffles in order --
        // the same additions in the same order as the general path below
        const bool valid = lane < E;
        const int r = valid ? st.row[lane] : INT_MAX;
        const unsigned vm = __ballot_sync(kFull, valid);
        const unsigned grp = __match_any_sync(kFull, r) & vm;
        const bool leader = valid && (__ffs(grp) - 1 == lane);
        const unsigned L = __ballot_sync(kFull, leader);
        M = __popc(L);
        int rank = 0;
        for (unsigned mm = L; mm; mm &= mm - 1) {
            const int rb = __shfl_sync(kFull, r, __ffs(mm) - 1);
            rank += (leader && rb < r) ? 1 : 0;
        }
        if (leader) {
            double lam = 0.0, phv = 0.0;
            for (unsigned gg = grp; gg; gg &= gg - 1) {
                const int e = __ffs(gg) - 1;
                lam = lam + st.prod[e];
                if (st.diag[e]) phv = st.ph[e];
            }
            st.rrow[rank] = r;
            st.rlam[rank] = lam;
            st.rphi[rank] = phv;
        }
        __syncwarp();
        // lane m now owns distinct row m (ascending)
        const bool hv = lane < M;
        const int row = hv ? st.rrow[lane] : 0;
        const double ph = hv ? st.rphi[lane] : 0.0, lm = hv ? st.rlam[lane] : 0.0;
        const bool in = hv && in_skeleton(ph, lm);
        const unsigned bpm = __ballot_sync(kFull, hv && ph != 0.0 && !in);
        const unsigned blm = __ballot_sync(kFull, hv && lm != 0.0 && !in);
        const int bpr = __shfl_sync(kFull, row, bpm ? 31 - __clz(bpm) : 0);   // the last such row
        const int blr = __shfl_sync(kFull, row, blm ? 31 - __clz(blm) : 0);
        if (bpm) g.bad_phi_row = bpr;
        if (blm) g.bad_lt_row = blr;
        const unsigned im = __ballot_sync(kFull, in);
        const double lh = (in && lm != 0.0) ? lm : 0.0;
        const double sq = in ? sqrt_skel(ph) : 0.0;
        g.n = __popc(im);
        if (im) {
            const int f0 = __ffs(im) - 1;
            g.first_row = __shfl_sync(kFull, row, f0);
            g.phi0 = __shfl_sync(kFull, ph, f0);
        }
        for (unsigned mm = im; mm; mm &= mm - 1) {   // ascending rows, sequential sums
            const int b = __ffs(mm) - 1;
            g.sl = g.sl + __shfl_sync(kFull, lh, b);
            g.sp = g.sp + __shfl_sync(kFull, ph, b);
            g.sr = g.sr + __shfl_sync(kFull, sq, b);
        }
        const Coef c = make_coef(g, p.cp, c_recip);
        bool nl = false;
        const double v = in ? update_entry_sq(row, ph, lh, sq, c, p.cp, nl) : 0.0;
        anynan = __any_sync(kFull, in && nl);
        double s = 0.0;
        for (unsigned mm = im; mm; mm &= mm - 1) s = s + __shfl_sync(kFull, v, __ffs(mm) - 1);
        const bool spos = s > 0.0;
        const double inv = 1.0 / (spos ? s : 1.0);
        const double nv = spos ? v * inv : v;
        const bool out = in && nv != 0.0;
        if (in) md = fabs(nv - ph);
        const unsigned om = __ballot_sync(kFull, out);
        const int pos = __popc(om & ((1u << lane) - 1u));
        cnt = __popc(om);
        if (hv) {
            st.rv[lane] = nv;
            st.rpos[lane] = out ? pos : -1;
        }
        bool mism = false;
        if (out) {
            if (row == 0) bm_new = nv;
            mism = pos >= co || hyb_row<T>(p.in, so, ao, pos) != row ||
                   !same_bits<T>(nv, hyb_val<T>(p.in, j, so, ao, pos));
        }
        changed = cnt != co || __any_sync(kFull, mism);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            md = fmax(md, __shfl_xor_sync(kFull, md, o));
            bm_new = bm_new + __shfl_xor_sync(kFull, bm_new, o);   // at most one nonzero term: exact
        }
    } else {
        // 2. rank by (row, staging order)
        for (int e = lane; e < E; e += 32) {
            const int r = st.row[e];
            int rank = 0;
            for (int f = 0; f < E; ++f) {
                const int rf = st.row[f];
                rank += (rf < r || (rf == r && f < e)) ? 1 : 0;
            }
            st.order[rank] = (short)e;
        }
        __syncwarp();
        // 3. one slot per distinct row: Lt in L order, PHI(r, j)
        for (int k0 = 0; k0 < E; k0 += 32) {
            const int k = k0 + lane;
            bool head = false;
            int r = 0;
            if (k < E) {
                r = st.row[st.order[k]];
                head = k == 0 || st.row[st.order[k - 1]] != r;
            }
            int tot;
            const int m = M + warp_excl_scan(head ? 1 : 0, lane, tot);
            if (head) {
                double lam = 0.0, phv = 0.0;
                for (int kk = k; kk < E; ++kk) {
                    const int e = st.order[kk];
                    if (st.row[e] != r) break;
                    lam = lam + st.prod[e];
                    if (st.diag[e]) phv = st.ph[e];
                }
                st.rrow[m] = r;
                st.rlam[m] = lam;
                st.rphi[m] = phv;
            }
            M += tot;
        }
        __syncwarp();
        // 4. skeleton, aggregates in ascending row order (every lane, from smem)
        for (int m = 0; m < M; ++m) {
            const double ph = st.rphi[m], lm = st.rlam[m];
            const bool in = in_skeleton(ph, lm);
            if (ph != 0.0 && !in) g.bad_phi_row = st.rrow[m];
            if (lm != 0.0 && !in) g.bad_lt_row = st.rrow[m];
            if (in) {
                if (g.n == 0) { g.first_row = st.rrow[m]; g.phi0 = ph; }
                g.n++;
                g.sl = g.sl + ((lm != 0.0) ? lm : 0.0);
                g.sp = g.sp + ph;
                g.sr = g.sr + sqrt_skel(ph);
            }
        }
        const Coef c = make_coef(g, p.cp, c_recip);
        bool nan = false;
        for (int m = lane; m < M; m += 32) {
            const double ph = st.rphi[m], lm = st.rlam[m];
            const bool in = in_skeleton(ph, lm);
            bool nl = false;
            const double v = update_entry(in ? st.rrow[m] : 1, in ? ph : 0.0, (in && lm != 0.0) ? lm : 0.0, c, p.cp, nl);
            st.rv[m] = in ? v : 0.0;
            nan |= in && nl;
        }
        __syncwarp();
        double s = 0.0;
        for (int m = 0; m < M; ++m)
            if (in_skeleton(st.rphi[m], st.rlam[m])) s = s + st.rv[m];
        const bool spos = s > 0.0;
        const double inv = 1.0 / (spos ? s : 1.0);
        // 5. normalise, output positions, the change test against the old column
        bool mism = false;
        for (int m0 = 0; m0 < M; m0 += 32) {
            const int m = m0 + lane;
            bool out = false;
            double nv = 0.0, ph = 0.0;
            int r = 0;
            if (m < M) {
                ph = st.rphi[m];
                r = st.rrow[m];
                const bool in = in_skeleton(ph, st.rlam[m]);
                nv = spos ? st.rv[m] * inv : st.rv[m];
                out = in && nv != 0.0;
                if (in) md = fmax(md, fabs(nv - ph));
                st.rv[m] = nv;
            }
            int tot;
            const int pos = cnt + warp_excl_scan(out ? 1 : 0, lane, tot);
            if (m < M) st.rpos[m] = out ? pos : -1;
            if (out) {
                if (r == 0) bm_new = nv;
                mism |= pos >= co || hyb_row<T>(p.in, so, ao, pos) != r || !same_bits<T>(nv, hyb_val<T>(p.in, j, so, ao, pos));
            }
            cnt += tot;
        }
        changed = cnt != co || __any_sync(kFull, mism);
        anynan = __any_sync(kFull, nan);
    #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            md = fmax(md, __shfl_xor_sync(kFull, md, o));
            bm_new = bm_new + __shfl_xor_sync(kFull, bm_new, o);   // at most one nonzero term: exact
        }
        __syncwarp();
    }
    __syncwarp();
    // 6. statistics, pool placement, emit, marks
    long long off = 0;
    if (lane == 0) {
        VRes res;
        vres_init(res);
        res.nan = anynan; res.bad_phi_row = g.bad_phi_row; res.bad_lt_row = g.bad_lt_row;
        report_flags(res, j, p);
        acc.md = fmax(acc.md, md);
        const int skc_old = skc_pre;
        acc.dn += cnt - (full ? 0 : co);
        acc.ds += g.n - skc_old;
        if (p.track && (full || g.n != skc_old)) p.ws.skc[jl] = g.n;
        if (cnt > 2) off = (!full && osig <= -cnt) ? (long long)oaux : pool_take(p, j, cnt, true);
        if (cnt == 0) {
            p.out.sig[j] = FT_SIG_EMPTY;
        } else if (cnt > 2 && off >= 0) {
            p.out.sig[j] = -cnt;
            p.out.aux[j] = (int)off;
        }
    }
    off = __shfl_sync(kFull, off, 0);
    __syncwarp();
    bool nf = false;
    for (int m = lane; m < M; m += 32) {
        const int pos = st.rpos[m];
        if (pos < 0) continue;
        const int r = st.rrow[m];
        const double nv = st.rv[m];
        nf |= !isfinite(nv);
        if (cnt <= 2) {
            if (pos == 0) {
                p.out.sig[j] = cnt == 2 ? (r | kPair) : r;
                ((T*)p.out.v0)[j] = (T)nv;
            } else {
                p.out.aux[j] = r;
                ((T*)p.out.v1)[j] = (T)nv;
            }
        } else if (off >= 0) {
            p.out.pidx[off + pos] = r;
            ((T*)p.out.pval)[off + pos] = (T)nv;
        }
    }
    if (nf) atomicOr(&p.ws.ctl->nonfinite, 1u);
    if (p.track && changed)
        for (int k = lane; k < n; k += 32) p.ws.stamp[pu >= 0 ? pu : __ldg(&p.lap_idx[q0 + k])] = nxt;
    const double bm_old = lane == 0 ? base_of<T>(p.in, j) : 0.0;
    __syncwarp();
    bm_fold(lane == 0 ? bm_new : 0.0, bm_old, full, s_bm);
}

template <typename T, bool UNIFORM, bool PACKED>
#ifndef FT_WIDE_MINB
#define FT_WIDE_MINB (1024 / FT_WIDE_TPB)      // 64 registers: 1024 threads per SM (both limits met, +1 % at C3)
#endif
__global__ void __launch_bounds__(kWideTPB, FT_WIDE_MINB) wide_kernel(const StepParams p) {
    pdl_wait();
    Control* ctl = p.ws.ctl;
    __shared__ long long s_bm[4];
    __shared__ double s_md[kWideWarps];
    __shared__ long long s_cnt[2 * kWideWarps];
    __shared__ WideStage s_st[kWideWarps];
    if (p.check_done && vload(&ctl->done)) return;
    // the four-row kernel's leftovers (wide[]), or all of the three-row
    // kernel's (w2[]) when there were too few for the four-row kernel
    const int n2 = vload(&ctl->n_w2);
    const bool direct = n2 < p.wide4_min;
    const int nc = direct ? n2 : vload(&ctl->n_w3);
    const int* list = direct ? p.ws.w2 : p.ws.wide;
    if ((int)blockIdx.x * kWideWarps >= nc) return;
    if (threadIdx.x < 4) s_bm[threadIdx.x] = 0;
    __syncthreads();
    const bool full = step_is_full(p);
    const unsigned char nxt = (unsigned char)(vload(&ctl->seq) + 1);
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int nw = gridDim.x * kWideWarps;
    Acc acc;
    acc_init(acc);
    for (int i = (blockIdx.x * kWideTPB + threadIdx.x) >> 5; i < nc; i += nw)
        staged_column<T, UNIFORM, PACKED>(p, __ldg(&list[i]), s_st[wi], full, nxt, lane, acc, s_bm);
    __syncthreads();
    acc_flush<kWideTPB>(acc, s_bm, s_md, s_cnt, ctl);
}

// the wide kernel's columns beyond its staging capacity (listed in act,
// which no kernel reads after the band kernel): one thread each, the exact
// windowed algorithm from global memory
constexpr int kDeepTPB = 32;

// the deep columns (listed in act by the warp kernel) by one warp, one lane
// each: run by the finalize kernel before its totals (they are rare -- none
// at C3-C5 -- and a kernel of their own cost a launch per step, ~1 %)
template <typename T, bool UNIFORM>
__device__ __forceinline__ void deep_pass(const StepParams& p) {
    Control* ctl = p.ws.ctl;
    __shared__ long long s_bm[4];
    __shared__ double s_md[1];
    __shared__ long long s_cnt[2];
    if (p.check_done && vload(&ctl->done)) return;
    const int nd = vload(&ctl->n_deep);
    if (nd == 0) return;                    // block-uniform
    if (threadIdx.x < 4) s_bm[threadIdx.x] = 0;
    __syncthreads();
    const bool full = step_is_full(p);
    const unsigned char nxt = (unsigned char)(vload(&ctl->seq) + 1);
    Acc acc;
    acc_init(acc);
    for (int i0 = 0; i0 < nd; i0 += kDeepTPB) {
        const int i = i0 + threadIdx.x;
        double bm_new = 0.0, bm_old = 0.0;
        if (i < nd) deep_column<T, UNIFORM>(p, __ldg(&p.ws.act[i]), full, nxt, acc, bm_new, bm_old);
        __syncwarp();
        bm_fold(bm_new, bm_old, full, s_bm);
    }
    __syncthreads();
    acc_flush<kDeepTPB>(acc, s_bm, s_md, s_cnt, ctl);   // thread 0's atomics precede its reads below
}

// ---------------------------------------------------------------------------
// finalize: the deep columns (one warp), then statistics record, error /
// convergence flags, the next step's mode, accumulator reset (one thread)

struct FinalizeParams {
    Workspace ws;
    ft_step_stats* trace;
    long long tiled_cap;  // capacity reported as the floor of `needed`
    int fixed_slot;       // 1: write trace[0] (single step), 0: trace[steps_done]
    int evolve;           // evolve mode: convergence / done handling (stop test
                          // parameters in the control block)
    int track;
    int out_id;           // the step's target buffer
    long long next_cap;   // pool capacity of the next step's target (this step's input)
};

template <typename T, bool UNIFORM>
__global__ void __launch_bounds__(kDeepTPB) finalize_kernel(const FinalizeParams f, const StepParams p) {
    pdl_wait();
    Control* ctl = f.ws.ctl;
    if (f.evolve && vload(&ctl->done)) return;
    deep_pass<T, UNIFORM>(p);
    if (threadIdx.x != 0) return;
    const bool full = !f.track || ctl->full != 0;
    long long nnz = ctl->acc_nnz, skel = ctl->acc_skel;
    long long bm[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) bm[k] = ctl->acc_bm[k];
    if (!full) {
        nnz += ctl->tot_nnz;
        skel += ctl->tot_skel;
#pragma unroll
        for (int k = 0; k < 4; ++k) bm[k] += ctl->tot_bm[k];
    }
    const int slot = f.fixed_slot ? 0 : ctl->steps_done;
    ft_step_stats st;
    st.max_delta = __longlong_as_double((long long)ctl->maxdelta_bits);
    st.base_mass = fx_value(bm);
    st.nnz_phi = nnz;
    st.nnz_skel = skel;
    st.nan_col = ctl->nan_key ? (int)(INT_MAX - ctl->nan_key) : -1;
    st.bad_col = -1; st.bad_row = -1; st.bad_is_lt = 0;
    const unsigned long long kp = ctl->bad_phi_key, kl = ctl->bad_lt_key;
    if (kp) { const unsigned long long k = ~kp; st.bad_col = (int)(k >> 32); st.bad_row = (int)(k & 0xffffffffULL); }
    else if (kl) { const unsigned long long k = ~kl; st.bad_col = (int)(k >> 32); st.bad_row = (int)(k & 0xffffffffULL); st.bad_is_lt = 1; }
    int status = FT_STATUS_OK;
    // the reference checks expand(PHI), expand(Lt), then NaN (field.py:238-250)
    if (st.bad_col >= 0) status = FT_STATUS_PATTERN;
    else if (st.nan_col >= 0) status = FT_STATUS_NAN;
    else if (ctl->overflow) status = FT_STATUS_OVERFLOW;
    const int stepno = ctl->steps_done + 1;
    st.step = stepno;
    long long need = (long long)ctl->pool_next[f.out_id];
    if (ctl->conv_next > need) need = ctl->conv_next;
    if (need < f.tiled_cap) need = f.tiled_cap;
    st.needed = need;
    bool converged = false;
    if (status == FT_STATUS_OK && f.evolve)
        converged = (st.max_delta < ctl->tol) && (st.base_mass < ctl->base_threshold);
    st.status = converged ? FT_STATUS_CONVERGED : status;
    f.trace[slot] = st;

    if (status == FT_STATUS_OK) {
        ctl->tot_nnz = nnz;
        ctl->tot_skel = skel;
#pragma unroll
        for (int k = 0; k < 4; ++k) ctl->tot_bm[k] = bm[k];
    }
    // the next step runs full when its target's pool is half used
    ctl->full = (!f.track || status != FT_STATUS_OK ||
                 2 * (long long)ctl->pool_next[f.out_id ^ 1] > f.next_cap) ? 1 : 0;
    ctl->seq = ctl->seq + 1;
    ctl->maxdelta_bits = 0ULL;
    ctl->bad_phi_key = 0ULL;
    ctl->bad_lt_key = 0ULL;
    ctl->acc_nnz = 0;
    ctl->acc_skel = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) ctl->acc_bm[k] = 0;
    ctl->nan_key = 0u;
    ctl->overflow = 0;
    ctl->n_act = 0;
    ctl->n_wide = 0;
    ctl->n_w2 = 0;
    ctl->n_w3 = 0;
    ctl->n_deep = 0;
    ctl->conv_next = 0;
    if (f.evolve) {
        if (status != FT_STATUS_OK) {
            ctl->done = 1;
            ctl->status = status;
            ctl->needed = st.needed;
        } else {
            ctl->steps_done = stepno;
            if (converged) { ctl->done = 1; ctl->status = FT_STATUS_CONVERGED; }
            else if (stepno >= ctl->max_steps) { ctl->done = 1; ctl->status = FT_STATUS_MAXSTEPS; }
        }
    }
}

// ---------------------------------------------------------------------------
// canonical CSC -> hybrid layout

template <typename T>
__global__ void __launch_bounds__(256) convert_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                      const T* __restrict__ val, int n, HybOut o, long long cap,
                                                      Control* ctl) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool active = j < n;
    int c0 = 0, cnt = 0;
    if (active) {
        c0 = __ldg(&ptr[j]);
        cnt = __ldg(&ptr[j + 1]) - c0;
    }
    const int need = cnt > 2 ? cnt : 0;
    int incl = need;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, s);
        if (lane >= s) incl += y;
    }
    const int wtot = __shfl_sync(kFull, incl, 31);
    long long base = 0;
    if (lane == 31 && wtot > 0) base = (long long)atomicAdd((unsigned long long*)&ctl->conv_next, (unsigned long long)wtot);
    base = __shfl_sync(kFull, base, 31);
    const bool fits = base + wtot <= cap;
    if (lane == 31 && !fits) atomicExch(&ctl->overflow, 1);
    if (!active) return;
    bool nf = false;
    if (cnt == 0) {
        o.sig[j] = FT_SIG_EMPTY;
    } else if (cnt <= 2) {
        const T x0 = val[c0];
        ((T*)o.v0)[j] = x0;
        nf |= !isfinite((double)x0);
        if (cnt == 1) {
            o.sig[j] = idx[c0];
        } else {
            const T x1 = val[c0 + 1];
            o.sig[j] = idx[c0] | kPair;
            o.aux[j] = idx[c0 + 1];
            ((T*)o.v1)[j] = x1;
            nf |= !isfinite((double)x1);
        }
    } else if (fits) {
        const long long off = base + incl - need;
        o.sig[j] = -cnt;
        o.aux[j] = (int)off;
        for (int t = 0; t < cnt; ++t) {
            o.pidx[off + t] = idx[c0 + t];
            const T x = val[c0 + t];
            ((T*)o.pval)[off + t] = x;
            nf |= !isfinite((double)x);
        }
    } else {
        o.sig[j] = FT_SIG_EMPTY;   // the step that follows reports the overflow
    }
    if (nf) atomicOr(&ctl->nonfinite, 1u);
}

// after a conversion: the next step is a full one, and neither buffer's pool
// may hand out the converted columns' entries
__global__ void convert_done_kernel(Control* ctl) {
    ctl->full = 1;
    ctl->pool_next[0] = (unsigned long long)ctl->conv_next;
    ctl->pool_next[1] = (unsigned long long)ctl->conv_next;
}

__global__ void convert_report_kernel(Control* ctl, ft_step_stats* st, long long cap) {
    st->status = ctl->overflow ? FT_STATUS_OVERFLOW : FT_STATUS_OK;
    st->needed = ctl->conv_next > cap ? ctl->conv_next : cap;
    ctl->overflow = 0;
    ctl->conv_next = 0;
}

// ---------------------------------------------------------------------------
// compaction: hybrid -> canonical CSC

struct CompactParams {
    int n_v;
    HybIn src[2];
    int sel;               // 0/1: source buffer; -1: pick by evolve parity
    int* out_ptr;
    int* out_idx;
    void* out_val;
    long long cap;
    Workspace ws;
    ft_step_stats* stats;  // single-step mode record (nullable)
    long long* control;    // evolve mode (nullable)
    int check_status;      // skip when stats->status reports a failed step
};

__device__ __forceinline__ int compact_source(const CompactParams& c) {
    if (c.check_status && c.stats && vload(&c.stats->status) != FT_STATUS_OK) return -1;
    if (c.sel >= 0) return c.sel;
    const int n = c.ws.ctl->steps_done;
    return n == 0 ? -1 : ((n & 1) ? 0 : 1);
}

constexpr int kCPT = FT_CCH / FT_CTPB;   // columns per thread (8)

__global__ void __launch_bounds__(FT_CTPB) compact_count_kernel(const CompactParams c) {
    __shared__ int s_scan[FT_CTPB / 32];
    const int src = compact_source(c);
    if (src < 0) return;
    const int* sig = c.src[src].sig;
    const int j0 = blockIdx.x * FT_CCH + threadIdx.x * kCPT;
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kCPT; ++k)
        if (j0 + k < c.n_v) sum += sig_count(__ldg(&sig[j0 + k]));
    int tot;
    block_excl_scan<FT_CTPB>(sum, s_scan, &tot);
    if (threadIdx.x == 0) c.ws.chunk_off[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) compact_scan_kernel(const CompactParams c) {
    __shared__ long long s_part[32];
    const int src = compact_source(c);
    const int nc = c.ws.num_chunks;
    const int tid = threadIdx.x;
    long long* off = c.ws.chunk_off;
    if (src < 0) {
        if (tid == 0 && c.control) { c.control[3] = 0; c.control[4] = 0; c.control[5] = 0; }
        return;
    }
    const int per = (nc + 1023) / 1024;
    const int b0 = tid * per;
    long long sum = 0;
    for (int k = 0; k < per; ++k)
        if (b0 + k < nc) sum += off[b0 + k];
    long long incl = sum;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_part[warp] = incl;
    __syncthreads();
    long long pre = 0, tot = 0;
    for (int k = 0; k < 32; ++k) {
        if (k < warp) pre += s_part[k];
        tot += s_part[k];
    }
    long long run = pre + incl - sum;
    for (int k = 0; k < per; ++k) {
        if (b0 + k < nc) {
            const long long v = off[b0 + k];
            off[b0 + k] = run;
            run += v;
        }
    }
    if (tid == 0) {
        off[nc] = tot;
        const bool fits = tot <= c.cap && tot <= (long long)INT_MAX;
        off[nc + 1] = fits ? 1 : 0;
        if (fits) c.out_ptr[c.n_v] = (int)tot;
        if (c.stats) {
            c.stats->nnz_phi = tot;
            if (!fits) { c.stats->status = FT_STATUS_OUT_OVERFLOW; c.stats->needed = tot; }
            else if (!c.check_status) c.stats->status = FT_STATUS_OK;
        }
        if (c.control) { c.control[3] = fits ? 1 : 2; c.control[4] = tot; c.control[5] = tot; }
    }
}

template <typename T>
__global__ void __launch_bounds__(FT_CTPB) compact_copy_kernel(const CompactParams c) {
    __shared__ int s_scan[FT_CTPB / 32];
    const int src = compact_source(c);
    if (src < 0) return;
    if (c.ws.chunk_off[c.ws.num_chunks + 1] == 0) return;  // does not fit
    const HybIn h = c.src[src];
    T* oval = (T*)c.out_val;
    const int j0 = blockIdx.x * FT_CCH + threadIdx.x * kCPT;
    int sg[kCPT];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
        sg[k] = (j0 + k < c.n_v) ? __ldg(&h.sig[j0 + k]) : FT_SIG_EMPTY;
        sum += sig_count(sg[k]);
    }
    int tot;
    const int pre = block_excl_scan<FT_CTPB>(sum, s_scan, &tot);
    long long o = c.ws.chunk_off[blockIdx.x] + pre;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
        if (j0 + k < c.n_v) {
            const int u = j0 + k;
            c.out_ptr[u] = (int)o;
            const int cnt = sig_count(sg[k]);
            const int a = cnt >= 2 ? __ldg(&h.aux[u]) : 0;
            for (int t = 0; t < cnt; ++t) {
                c.out_idx[o + t] = hyb_row<T>(h, sg[k], a, t);
                oval[o + t] = (T)hyb_val<T>(h, u, sg[k], a, t);
            }
            o += cnt;
        }
    }
}

__global__ void evolve_reset_kernel(Control* ctl, int max_steps, double tol, double thr) {
    ctl->nonfinite = 0u;    // ft_tiled_from_csc raises it again for non-finite input
    ctl->max_steps = max_steps;
    ctl->tol = tol;
    ctl->base_threshold = thr;
    ctl->done = 0;
    ctl->steps_done = 0;
    ctl->status = FT_STATUS_OK;
    ctl->needed = 0;
}

__global__ void evolve_report_kernel(const Control* ctl, long long* control) {
    control[0] = ctl->steps_done;
    control[1] = ctl->status;
    control[2] = ctl->needed;
}

__global__ void nonfinite_reset_kernel(Control* ctl) { ctl->nonfinite = 0u; }

// ---------------------------------------------------------------------------
// packed L^T neighbour table (FT_LAP_PACKED)

__global__ void lap_pack_kernel(const int* __restrict__ ptr, const int* __restrict__ idx, int n_cols,
                                int col_base, int4* __restrict__ pack, int* n_csr) {
    const int jl = blockIdx.x * blockDim.x + threadIdx.x;
    if (jl >= n_cols) return;
    const int q0 = ptr[jl], n = ptr[jl + 1] - q0;
    const long long j = (long long)col_base + jl;
    int s[kMD];
    bool ok = n >= 1 && n <= kMD;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        s[k] = kPackEmpty;
        if (ok && k < n) {
            const long long dl = (long long)idx[q0 + k] - j;
            if (dl < -32767 || dl > 32767) ok = false;
            else s[k] = (int)dl;
        }
    }
    if (!ok) {
#pragma unroll
        for (int k = 0; k < kMD; ++k) s[k] = kPackEmpty;
        atomicAdd(n_csr, 1);
    }
    int w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = (s[2 * q] & 0xffff) | (s[2 * q + 1] << 16);
    pack[jl] = make_int4(w[0], w[1], w[2], w[3]);
}

typedef void (*StepKernelFn)(const StepParams);

#define FT_PICK3(K, dtype, uni, packed)                                               \
    ((dtype) == FT_F64 ? ((uni) ? ((packed) ? K<double, true, true> : K<double, true, false>) \
                                : K<double, false, false>)                             \
                       : ((uni) ? ((packed) ? K<float, true, true> : K<float, true, false>)   \
                                : K<float, false, false>))
#define FT_PICK2(K, dtype, uni)                                                              \
    ((dtype) == FT_F64 ? ((uni) ? K<double, true> : K<double, false>) : ((uni) ? K<float, true> : K<float, false>))

}  // namespace ft

// ---------------------------------------------------------------------------
// C ABI

static thread_local char g_err[512] = "";

static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

static int cuda_check(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
        return FT_ERR_CUDA;
    }
    return FT_OK;
}

extern "C" int ft_abi_version(void) { return FT_ABI_VERSION; }
extern "C" const char* ft_last_error(void) { return g_err; }

extern "C" size_t ft_workspace_bytes(int32_t n_vertices) {
    return ft::workspace_bytes(n_vertices < 0 ? 0 : n_vertices);
}

extern "C" int ft_workspace_init(void* workspace, size_t bytes, void* stream) {
    if (!workspace) return set_err(FT_ERR_ARG, "null workspace");
    cudaMemsetAsync(workspace, 0, bytes, (cudaStream_t)stream);
    return cuda_check("ft_workspace_init");
}

static int check_tiled(const ft_tiled* t, int n_rows, int n_cols) {
    if (!t || !t->sig || !t->aux || !t->v0 || !t->v1) return set_err(FT_ERR_ARG, "null hybrid buffer");
    if (n_rows < 1 || n_rows > FT_SIG_PAIR)
        return set_err(FT_ERR_SHAPE, "the hybrid layout holds at most 2^30 layer rows");
    if (t->capacity < 0 || t->capacity > (int64_t)INT_MAX) return set_err(FT_ERR_ARG, "pool capacity out of range");
    if (t->capacity > 0 && (!t->pool_idx || !t->pool_val)) return set_err(FT_ERR_ARG, "null pool");
    if (t->n_rows != n_rows || t->n_cols != n_cols) return set_err(FT_ERR_SHAPE, "hybrid buffer has wrong shape");
    return FT_OK;
}

// Per-device state (a process may drive several GPUs, one host thread per
// device at a time): whether c_recip is set on the device, the SM count, the
// per-kernel grid sizes, the graph stream and the evolve-graph cache (with
// its own lock).  Indexed by the current device ordinal.
struct GraphKey {
    const void* ptrs[18];
    long long caps[3];
    double prm[8];
    int ints[6];
    bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};

struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    bool used;
};

struct DevState {
    std::mutex mu;
    int init;
    int sms;
    int band_grid[2][2][2];
    cudaStream_t gstream;
    cudaEvent_t gev[2];
    GraphEntry graphs[8];
    int graph_next;
    cudaEvent_t pev[7];       // ft_step_phases: phase boundaries (timing events)
};
static DevState g_dev[64];

static DevState& dev_state() {
    int d = 0;
    cudaGetDevice(&d);
    return g_dev[d & 63];
}

static int pdl_enabled() {
    static const int on = [] {
        const char* e = getenv("FT_PDL");
        return e ? atoi(e) : 1;
    }();
    return on;
}

// launch k on s, programmatically dependent on the stream's previous kernel
// (its launch and CTA ramp overlap the predecessor's tail; the kernel's
// pdl_wait() orders every memory access after the predecessor)
static int trace_launches() {
    static const int on = [] {
        const char* e = getenv("FT_TRACE");
        return e ? atoi(e) : 0;
    }();
    return on;
}

template <typename... KA, typename... AA>
static void launch_dep(void (*k)(KA...), int grid, int block, cudaStream_t s, AA&&... args) {
    if (trace_launches()) fprintf(stderr, "[ft] launch %p grid %d block %d\n", (void*)k, grid, block);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    if (pdl_enabled()) { cfg.attrs = at; cfg.numAttrs = 1; }
    cudaLaunchKernelEx(&cfg, k, std::forward<AA>(args)...);
}

static void lib_init() {
    DevState& d = dev_state();
    if (d.init) return;
    std::lock_guard<std::mutex> lk(d.mu);
    if (d.init) return;
    double h[33];
    h[0] = 0.0;
    for (int n = 1; n <= 32; ++n) h[n] = 1.0 / (double)n;
    cudaMemcpyToSymbol(ft::c_recip, h, sizeof(h));
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        sms = 148;
    d.sms = sms;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int c = 0; c < 2; ++c) {
                const ft::StepKernelFn k = FT_PICK3(ft::band_kernel, a ? FT_F32 : FT_F64, b, b && c);
                int per_sm = 0;
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, ft::kBandTPB, 0) != cudaSuccess ||
                    per_sm < 1)
                    per_sm = 4;
                d.band_grid[a][b][c] = per_sm * sms;
            }
    cudaGetLastError();
    d.init = 1;
}

// One step's column kernels (prep, band, wide3, wide) on s; dom == nullptr:
// the whole field, otherwise the owned column range of a partitioned field
// (lap_t then holds the owned columns of L^T only and the workspace is sized
// for the owned columns; every step is a full step).
// `keep` receives the step's parameters (the finalize kernel's deep pass
// reads them); launch == false only validates and fills them.
static int launch_columns(const ft_csc* lap_t, int32_t lap_flags, const ft_tiled* in, ft_tiled* out, int out_id,
                          int32_t dtype, const ft_params* prm, void* workspace, size_t ws_bytes, int check_done,
                          cudaStream_t s, const ft_domain* dom = nullptr, const cudaEvent_t* ev = nullptr,
                          ft::StepParams* keep = nullptr, bool launch = true) {
    if (!lap_t || !out || !in || !prm || !workspace) return set_err(FT_ERR_ARG, "null argument");
    if (dtype != FT_F64 && dtype != FT_F32) return set_err(FT_ERR_ARG, "bad dtype");
    const int n_rows = in->n_rows, n_v = in->n_cols;
    if (n_v <= 0) return set_err(FT_ERR_SHAPE, "empty field");
    const int j_base = dom ? dom->col_begin : 0;
    const int n_own = dom ? dom->col_count : n_v;
    if (dom && (j_base < 0 || n_own < 1 || (long long)j_base + n_own > n_v))
        return set_err(FT_ERR_SHAPE, "domain outside the field");
    if (lap_t->n_rows != n_v || lap_t->n_cols != n_own)
        return set_err(FT_ERR_SHAPE, "Laplacian size does not match field");
    int rc = check_tiled(in, n_rows, n_v);
    if (rc == FT_OK) rc = check_tiled(out, n_rows, n_v);
    if (rc != FT_OK) return rc;
    const long long step_cap = dom ? dom->step_capacity : out->capacity;
    if (step_cap < 0 || step_cap > out->capacity) return set_err(FT_ERR_ARG, "domain step capacity out of range");
    if (ws_bytes < ft::workspace_bytes(n_v)) return set_err(FT_ERR_ARG, "workspace too small");
    if (out_id != 0 && out_id != 1) return set_err(FT_ERR_ARG, "out_id must be 0 or 1");
    ft::StepParams p;
    p.n_v = n_own;
    p.j_base = j_base;
    p.lap_ptr = lap_t->col_ptr;
    p.lap_idx = lap_t->row_idx;
    p.lap_val = lap_t->values;
    p.in = ft::hyb_in(in);
    p.out = ft::hyb_out(out);
    p.cap = step_cap;
    p.out_id = out_id;
    p.cp.w = prm->w; p.cp.a = prm->a; p.cp.e = prm->e; p.cp.eb = prm->e_base; p.cp.mu = prm->mu; p.cp.dt = prm->dt;
    p.cp.finite = std::isfinite(p.cp.w) && std::isfinite(p.cp.a) && std::isfinite(p.cp.e) &&
                  std::isfinite(p.cp.eb) && std::isfinite(p.cp.mu) && std::isfinite(p.cp.dt);
    p.ws = ft::carve_workspace(workspace, n_v);      // the buffer's columns (owned + halo in a domain)
    p.check_done = check_done;
    p.track = (lap_flags & FT_LAP_SYMMETRIC) ? 1 : 0;
    const bool uni = (lap_flags & FT_LAP_UNIFORM) != 0;
    const bool packed = uni && (lap_flags & FT_LAP_PACKED) != 0;
    p.lap_pack = packed ? (const int4*)lap_t->values : nullptr;
    p.force_check = (lap_flags & FT_LAP_CHECK_FINITE) != 0;
    p.report_ids = dom ? dom->report_ids : nullptr;
    const char* w4 = getenv("FT_WIDE4_MIN");     // tests: exercise the four-row kernel on small fields
    p.wide4_min = w4 ? atoi(w4) : ft::kWide4Min;
    // the four-row kernel only under a hint (a dense band, or a young field
    // whose band is still forming): otherwise it is a no-op launch below its
    // threshold (C3 steady state +1.9 % without it) and the warp kernel takes
    // every three-row leftover directly
    const bool run_w4 = (lap_flags & (FT_HINT_DENSE_BAND | FT_HINT_FOUR_ROW)) || w4;
    if (!run_w4) p.wide4_min = INT_MAX;
    lib_init();
    if (keep) *keep = p;
    if (!launch) return FT_OK;
    DevState& d = dev_state();
    const char* kenv = getenv("FT_KERNELS");   // debug: bit mask of the column kernels to launch
    const int kmask = kenv ? atoi(kenv) : 15;
    const int prep_span = n_own + (j_base & 15);  // 16-byte aligned tiles from j_base & ~15
    const int prep_grid = (prep_span + ft::kPrepCols * ft::kPrepTPB - 1) / (ft::kPrepCols * ft::kPrepTPB);
    if (kmask & 1) launch_dep(ft::prep_kernel, prep_grid, ft::kPrepTPB, s, p);
    if (ev) cudaEventRecord(ev[0], s);
    int bg = d.band_grid[dtype == FT_F32][uni][packed];
    const int need_b = (n_own + ft::kBandTPB - 1) / ft::kBandTPB;
    if (bg > need_b) bg = need_b;
    if (kmask & 2) launch_dep(FT_PICK3(ft::band_kernel, dtype, uni, packed), bg, ft::kBandTPB, s, p);
    if (ev) cudaEventRecord(ev[1], s);
    if (kmask & 4) {
        if (lap_flags & FT_HINT_DENSE_BAND)
            launch_dep(FT_PICK3(ft::wide3_dense_kernel, dtype, uni, packed), ft::kWide3DenseMinB * d.sms,
                       ft::kWide3TPB, s, p);
        else
            launch_dep(FT_PICK3(ft::wide3_kernel, dtype, uni, packed), FT_W3_MINB * d.sms, ft::kWide3TPB, s, p);
    }
    if (ev) cudaEventRecord(ev[2], s);
    if (kmask & 8) {
        if (run_w4)
            launch_dep(FT_PICK3(ft::wide4_kernel, dtype, uni, packed), FT_W4_MINB * d.sms, ft::kWide4TPB, s, p);
        launch_dep(FT_PICK3(ft::wide_kernel, dtype, uni, packed), FT_WIDE_MINB * d.sms, ft::kWideTPB, s, p);
    }
    if (ev) cudaEventRecord(ev[3], s);
    return cuda_check("step kernels");
}

// the finalize kernel (with the deep pass of the step `p`, launched by
// launch_columns with the same arguments)
static void launch_finalize(const ft::Workspace& ws, ft_step_stats* trace, long long tiled_cap, int evolve,
                            int lap_flags, int out_id, long long next_cap, bool domain, cudaStream_t s,
                            const ft::StepParams& p, int32_t dtype) {
    ft::FinalizeParams f;
    f.ws = ws; f.trace = trace; f.tiled_cap = tiled_cap; f.fixed_slot = evolve ? 0 : 1;
    f.evolve = evolve;
    f.track = (lap_flags & FT_LAP_SYMMETRIC) ? 1 : 0;
    (void)domain;
    f.out_id = out_id;
    f.next_cap = next_cap;
    const bool uni = (lap_flags & FT_LAP_UNIFORM) != 0;
    launch_dep(FT_PICK2(ft::finalize_kernel, dtype, uni), 1, ft::kDeepTPB, s, f, p);
}

static int launch_convert(const ft_csc* src, ft_tiled* dst, int32_t dtype, const ft::Workspace& ws,
                          cudaStream_t s) {
    if (!src || !src->col_ptr || (!src->row_idx && src->capacity > 0)) return set_err(FT_ERR_ARG, "null argument");
    if (dtype != FT_F64 && dtype != FT_F32) return set_err(FT_ERR_ARG, "bad dtype");
    int rc = check_tiled(dst, src->n_rows, src->n_cols);
    if (rc != FT_OK) return rc;
    const int n = src->n_cols;
    if (n <= 0) return set_err(FT_ERR_SHAPE, "empty field");
    const int grid = (n + 255) / 256;
    if (dtype == FT_F64)
        ft::convert_kernel<double><<<grid, 256, 0, s>>>(src->col_ptr, src->row_idx, (const double*)src->values, n,
                                                       ft::hyb_out(dst), dst->capacity, ws.ctl);
    else
        ft::convert_kernel<float><<<grid, 256, 0, s>>>(src->col_ptr, src->row_idx, (const float*)src->values, n,
                                                      ft::hyb_out(dst), dst->capacity, ws.ctl);
    ft::convert_done_kernel<<<1, 1, 0, s>>>(ws.ctl);
    return cuda_check("ft_tiled_from_csc");
}

static int launch_compact(ft::CompactParams& c, int dtype, cudaStream_t s) {
    const int nc = c.ws.num_chunks;
    ft::compact_count_kernel<<<nc, FT_CTPB, 0, s>>>(c);
    ft::compact_scan_kernel<<<1, 1024, 0, s>>>(c);
    if (dtype == FT_F64) ft::compact_copy_kernel<double><<<nc, FT_CTPB, 0, s>>>(c);
    else ft::compact_copy_kernel<float><<<nc, FT_CTPB, 0, s>>>(c);
    return cuda_check("compact");
}

extern "C" int ft_tiled_from_csc(const ft_csc* src, ft_tiled* dst, int32_t dtype, void* workspace,
                                 size_t ws_bytes, ft_step_stats* stats, void* stream) {
    if (!src || !dst || !workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (ws_bytes < ft::workspace_bytes(src->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const ft::Workspace ws = ft::carve_workspace(workspace, src->n_cols);
    const int rc = launch_convert(src, dst, dtype, ws, s);
    if (rc != FT_OK) return rc;
    ft::convert_report_kernel<<<1, 1, 0, s>>>(ws.ctl, stats, dst->capacity);
    return cuda_check("ft_tiled_from_csc");
}

extern "C" int ft_step_run(const ft_csc* lap_t, int32_t lap_flags, const ft_tiled* in, ft_tiled* out,
                           int32_t out_id, int32_t dtype, const ft_params* params, void* workspace,
                           size_t ws_bytes, int32_t phases, ft_step_stats* stats, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (phases & FT_PHASE_COLUMNS) {
        const int rc = launch_columns(lap_t, lap_flags, in, out, out_id, dtype, params, workspace, ws_bytes, 0, s);
        if (rc != FT_OK) return rc;
    }
    if (phases & FT_PHASE_FINALIZE) {
        if (!stats || !in || !out || !workspace) return set_err(FT_ERR_ARG, "null argument");
        if (ws_bytes < ft::workspace_bytes(in->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
        ft::StepParams p;
        const int rc = launch_columns(lap_t, lap_flags, in, out, out_id, dtype, params, workspace, ws_bytes, 0, s,
                                      nullptr, nullptr, &p, false);
        if (rc != FT_OK) return rc;
        launch_finalize(ft::carve_workspace(workspace, in->n_cols), stats, out->capacity, 0, lap_flags, out_id,
                        in->capacity, false, s, p, dtype);
    }
    return cuda_check("ft_step_run");
}

static void fill_compact(ft::CompactParams& c, const ft_tiled* a, const ft_tiled* b, int sel, ft_csc* dst,
                         void* workspace) {
    c.n_v = dst->n_cols;
    c.src[0] = ft::hyb_in(a);
    c.src[1] = ft::hyb_in(b ? b : a);
    c.sel = sel;
    c.out_ptr = dst->col_ptr; c.out_idx = dst->row_idx; c.out_val = dst->values; c.cap = dst->capacity;
    c.ws = ft::carve_workspace(workspace, dst->n_cols);
    c.stats = nullptr;
    c.control = nullptr;
    c.check_status = 0;
}

extern "C" int ft_compact(const ft_tiled* src, ft_csc* dst, int32_t dtype, void* workspace, size_t ws_bytes,
                          ft_step_stats* stats, void* stream) {
    if (!src || !dst || !workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (src->n_cols != dst->n_cols || src->n_rows != dst->n_rows) return set_err(FT_ERR_SHAPE, "shape mismatch");
    if (ws_bytes < ft::workspace_bytes(dst->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    if (dst->n_cols == 0) return set_err(FT_ERR_SHAPE, "empty field");
    ft::CompactParams c;
    fill_compact(c, src, nullptr, 0, dst, workspace);
    c.stats = stats;
    return launch_compact(c, dtype, (cudaStream_t)stream);
}

static int step_impl(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in, ft_tiled* scratch_in,
                     ft_tiled* scratch_out, ft_csc* phi_out, int32_t dtype, const ft_params* params,
                     void* workspace, size_t ws_bytes, ft_step_stats* stats, cudaStream_t s, float* phase_ms) {
    if (!phi_in || !phi_out || !stats || !scratch_in || !scratch_out) return set_err(FT_ERR_ARG, "null argument");
    if (phi_out->n_cols != phi_in->n_cols || phi_out->n_rows != phi_in->n_rows)
        return set_err(FT_ERR_SHAPE, "output buffer has wrong shape");
    if (ws_bytes < ft::workspace_bytes(phi_in->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    const cudaEvent_t* ev = nullptr;
    if (phase_ms) {
        DevState& d = dev_state();
        std::lock_guard<std::mutex> lk(d.mu);
        if (!d.pev[0])
            for (int k = 0; k < 7; ++k)
                if (cudaEventCreate(&d.pev[k]) != cudaSuccess) return set_err(FT_ERR_CUDA, "event create");
        ev = d.pev;
        cudaEventRecord(ev[0], s);
    }
    ft::Workspace ws = ft::carve_workspace(workspace, phi_in->n_cols);
    ft::nonfinite_reset_kernel<<<1, 1, 0, s>>>(ws.ctl);
    int rc = launch_convert(phi_in, scratch_in, dtype, ws, s);
    if (rc != FT_OK) return rc;
    ft::StepParams p;
    rc = launch_columns(lap_t, lap_flags, scratch_in, scratch_out, 0, dtype, params, workspace, ws_bytes, 0, s,
                        nullptr, ev ? ev + 1 : nullptr, &p);
    if (rc != FT_OK) return rc;
    const long long cap = scratch_out->capacity < scratch_in->capacity ? scratch_out->capacity : scratch_in->capacity;
    launch_finalize(ws, stats, cap, 0, lap_flags, 0, scratch_in->capacity, false, s, p, dtype);
    // the compaction always runs; the host ignores it if the step failed
    ft::CompactParams c;
    fill_compact(c, scratch_out, nullptr, 0, phi_out, workspace);
    c.stats = stats;
    c.check_status = 1;
    rc = launch_compact(c, dtype, s);
    if (rc != FT_OK || !ev) return rc;
    cudaEventRecord(ev[5], s);
    if (cudaEventSynchronize(ev[5]) != cudaSuccess) return set_err(FT_ERR_CUDA, "phase timing");
    // ev: 0 start | convert + prep | 1 | band | 2 | wide3 | 3 | wide4 + wide | 4 | finalize (+ deep) + compact | 5
    for (int k = 0; k < 5; ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
        phase_ms[k] = ms;
    }
    return cuda_check("ft_step_phases");
}

extern "C" int ft_step(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in, ft_tiled* scratch_in,
                       ft_tiled* scratch_out, ft_csc* phi_out, int32_t dtype, const ft_params* params,
                       void* workspace, size_t ws_bytes, ft_step_stats* stats, void* stream) {
    return step_impl(lap_t, lap_flags, phi_in, scratch_in, scratch_out, phi_out, dtype, params, workspace, ws_bytes,
                     stats, (cudaStream_t)stream, nullptr);
}

extern "C" int ft_step_phases(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in, ft_tiled* scratch_in,
                              ft_tiled* scratch_out, ft_csc* phi_out, int32_t dtype, const ft_params* params,
                              void* workspace, size_t ws_bytes, ft_step_stats* stats, float* phase_ms,
                              void* stream) {
    if (!phase_ms) return set_err(FT_ERR_ARG, "null argument");
    return step_impl(lap_t, lap_flags, phi_in, scratch_in, scratch_out, phi_out, dtype, params, workspace, ws_bytes,
                     stats, (cudaStream_t)stream, phase_ms);
}

// The steady part of evolve (steps 2, 3, ...: a -> b, b -> a) repeats with
// period 2, so kGraphSteps steps are captured once into a CUDA graph and
// replayed; steps past max_steps / convergence / a failure are device-side
// no-ops (every kernel tests the done flag).  Graphs are cached per device
// by their launch configuration (buffers, couplings, flags -- the stop test
// lives in the control block, so one graph serves every max_steps / tol).
constexpr int kGraphSteps = 16;

static int graph_stream_init(DevState& d) {
    if (d.gstream) return FT_OK;
    if (cudaStreamCreateWithFlags(&d.gstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.gev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.gev[1], cudaEventDisableTiming) != cudaSuccess) {
        d.gstream = nullptr;
        return FT_ERR_CUDA;
    }
    return FT_OK;
}

extern "C" int ft_evolve(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in, ft_tiled* work_a,
                         ft_tiled* work_b, ft_csc* phi_out, int32_t dtype, const ft_params* params,
                         int32_t max_steps, double tol, double base_threshold, void* workspace,
                         size_t ws_bytes, ft_step_stats* trace, int64_t* control, void* stream) {
    if (!phi_in || !phi_out || !work_a || !work_b || !trace || !control)
        return set_err(FT_ERR_ARG, "null argument");
    if (max_steps < 1) return set_err(FT_ERR_SHAPE, "max_steps must be >= 1");
    if (phi_out->n_cols != phi_in->n_cols || phi_out->n_rows != phi_in->n_rows)
        return set_err(FT_ERR_SHAPE, "output buffer has wrong shape");
    if (ws_bytes < ft::workspace_bytes(phi_in->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    ft::Workspace ws = ft::carve_workspace(workspace, phi_in->n_cols);
    lib_init();
    DevState& d = dev_state();
    // step i (0-based) writes a (buffer 0) when i is even, b (buffer 1) when odd
    auto step = [&](int i, cudaStream_t ms) -> int {
        ft_tiled* out = (i & 1) ? work_b : work_a;
        const ft_tiled* in_t = (i & 1) ? work_a : work_b;
        ft::StepParams p;
        const int r = launch_columns(lap_t, lap_flags, in_t, out, i & 1, dtype, params, workspace, ws_bytes, 1, ms,
                                     nullptr, nullptr, &p);
        if (r != FT_OK) return r;
        launch_finalize(ws, trace, out->capacity, 1, lap_flags, i & 1, in_t->capacity, false, ms, p, dtype);
        return FT_OK;
    };
    ft::evolve_reset_kernel<<<1, 1, 0, s>>>(ws.ctl, max_steps, tol, base_threshold);
    // canonical input -> b, step 1: b -> a
    int rc = launch_convert(phi_in, work_b, dtype, ws, s);
    if (rc != FT_OK) return rc;
    rc = step(0, s);
    if (rc != FT_OK) return rc;
    const int rest = max_steps - 1;
    static const int use_graph = [] {
        const char* e = getenv("FT_GRAPH");
        return e ? atoi(e) : 1;
    }();
    if (!use_graph) {
        for (int i = 1; i < max_steps; ++i) {
            rc = step(i, s);
            if (rc != FT_OK) return rc;
        }
    } else if (rest > 0) {
        GraphKey k;
        memset(&k, 0, sizeof(k));
        const void* ptrs[18] = {lap_t->col_ptr, lap_t->row_idx, lap_t->values, work_a->sig, work_a->aux,
                                work_a->v0, work_a->v1, work_a->pool_idx, work_a->pool_val, work_b->sig,
                                work_b->aux, work_b->v0, work_b->v1, work_b->pool_idx, work_b->pool_val,
                                workspace, trace, nullptr};
        memcpy(k.ptrs, ptrs, sizeof(ptrs));
        k.caps[0] = work_a->capacity; k.caps[1] = work_b->capacity; k.caps[2] = (long long)ws_bytes;
        const double prm[8] = {params->w, params->a, params->e, params->e_base, params->mu, params->dt, 0.0, 0.0};
        memcpy(k.prm, prm, sizeof(prm));
        const char* w4 = getenv("FT_WIDE4_MIN");     // baked into the captured launches
        const int ints[6] = {lap_flags, dtype, w4 ? atoi(w4) : ft::kWide4Min, phi_in->n_cols, phi_in->n_rows,
                             pdl_enabled()};
        memcpy(k.ints, ints, sizeof(ints));
        std::lock_guard<std::mutex> lk(d.mu);   // the graph cache and the graph stream
        if (graph_stream_init(d) != FT_OK) return cuda_check("ft_evolve(graph stream)");
        cudaStream_t gs = d.gstream;
        cudaEventRecord(d.gev[0], s);
        cudaStreamWaitEvent(gs, d.gev[0], 0);
        cudaGraphExec_t exec = nullptr;
        for (auto& e : d.graphs)
            if (e.used && e.key == k) exec = e.exec;
        if (!exec) {
            cudaGraph_t graph;
            if (cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
                return cuda_check("ft_evolve(begin capture)");
            for (int i = 1; i <= kGraphSteps; ++i) {
                const int r2 = step(i, gs);
                if (r2 != FT_OK) rc = r2;
            }
            const cudaError_t ec = cudaStreamEndCapture(gs, &graph);
            if (ec != cudaSuccess || rc != FT_OK) return rc != FT_OK ? rc : cuda_check("ft_evolve(end capture)");
            if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
                cudaGraphDestroy(graph);
                return cuda_check("ft_evolve(instantiate)");
            }
            cudaGraphDestroy(graph);
            // evict round robin; an exec is only ever launched under the lock
            GraphEntry& e = d.graphs[d.graph_next];
            d.graph_next = (d.graph_next + 1) % 8;
            if (e.used) cudaGraphExecDestroy(e.exec);
            e.key = k;
            e.exec = exec;
            e.used = true;
        }
        for (int done = 0; done < rest; done += kGraphSteps) cudaGraphLaunch(exec, gs);
        cudaEventRecord(d.gev[1], gs);
        cudaStreamWaitEvent(s, d.gev[1], 0);
    }
    ft::evolve_report_kernel<<<1, 1, 0, s>>>(ws.ctl, (long long*)control);
    ft::CompactParams c;
    fill_compact(c, work_a, work_b, -1, phi_out, workspace);
    c.control = (long long*)control;
    return launch_compact(c, dtype, s);
}

// ---------------------------------------------------------------------------
// partitioned field: one step of the owned columns (the halo kernels and the
// combine live in ft_domain.cu)

extern "C" int ft_domain_step(const ft_csc* lap_rows, int32_t lap_flags, const ft_tiled* in, ft_tiled* out,
                              int32_t dtype, const ft_params* params, const ft_domain* dom, void* workspace,
                              size_t ws_bytes, ft_step_stats* record, void* stream) {
    if (!in || !dom || !record) return set_err(FT_ERR_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int out_id = dom->out_id & 1;
    ft::StepParams p;
    const int rc = launch_columns(lap_rows, lap_flags, in, out, out_id, dtype, params, workspace, ws_bytes, 1, s,
                                  dom, nullptr, &p);
    if (rc != FT_OK) return rc;
    launch_finalize(ft::carve_workspace(workspace, in->n_cols), record, dom->step_capacity, 0, lap_flags, out_id,
                    dom->step_capacity, true, s, p, dtype);
    return cuda_check("ft_domain_step");
}

extern "C" int ft_laplacian_pack(const ft_csc* lap_t, int32_t col_base, int16_t* pack, int32_t* n_csr,
                                 void* stream) {
    if (!lap_t || !pack || !n_csr) return set_err(FT_ERR_ARG, "null argument");
    if (((uintptr_t)pack) & 15) return set_err(FT_ERR_ARG, "pack must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(n_csr, 0, sizeof(int32_t), s);
    const int n = lap_t->n_cols;
    if (n > 0) ft::lap_pack_kernel<<<(n + 255) / 256, 256, 0, s>>>(lap_t->col_ptr, lap_t->row_idx, n, col_base,
                                                                   (int4*)pack, n_csr);
    return cuda_check("ft_laplacian_pack");
}
