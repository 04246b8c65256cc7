// K12: the (1+1) EA's mutation draw on the device -- the random stream of
// the reference's loop (heuristics.py:318-325: for every child, for every
// position, `rng.random() < p` and on a hit `rng.integers(n_dev)`), for
// many independent chains at once (one CTA per chain), as the CSR lists
// the EA accept-chain kernel (K9) consumes.
//
// numpy's Generator(PCG64) is a 128-bit LCG with an XSL-RR output; its
// random() takes one whole 64-bit word and leaves the 32-bit buffer alone,
// integers(n) (n <= 2^32) is Lemire's method on 32-bit draws that take the
// buffered upper half of the previous word when one is cached (rng.py has
// the host restatement the tests pin against numpy). Almost every word is a
// random() miss, so the stream splits into
//   * a parallel phase: per block of T x W words, thread t jumps the LCG
//     ahead to word t*W (Brown's O(log n) jump), generates its W words (+1
//     to peek at the word after its last one) and records the hits
//     `w < lim` (lim = ceil(p * 2^53) << 11, i.e. (w >> 11) * 2^-53 < p)
//     with the word that follows each hit;
//   * a sequential walk over the block's hits (thread 0, about T*W/V of
//     them): misses between hits only advance (child, position); at a hit
//     the integers() draw takes the cached half or the next word, which is
//     then not a random() draw.
// Lemire's rejection branch (probability < n/2^32) and list overflow are
// reported per chain (status 2 / 1) and the host redraws that chain with
// rng.py; the result is then the reference's stream exactly either way.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/hetsched_b200.h"

namespace hs {
int set_error(int code, const std::string &msg);
}

namespace {

constexpr int kT = 256;  // threads per chain
constexpr int kW = 16;   // words per thread per block

struct U128 {
    uint64_t lo, hi;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

__device__ __forceinline__ U128 pcg_mult() {
    return U128{4865540595714422341ull, 2549297995355413924ull};
}

// (mult, plus) with state_{k+n} = mult * state_k + plus (Brown 1994)
__device__ void lcg_jump(uint64_t n, U128 inc, U128 &mult, U128 &plus) {
    U128 am{1, 0}, ap{0, 0}, cm = pcg_mult(), cp = inc;
    while (n) {
        if (n & 1) {
            am = mul128(am, cm);
            ap = add128(mul128(ap, cm), cp);
        }
        cp = mul128(add128(cm, U128{1, 0}), cp);
        cm = mul128(cm, cm);
        n >>= 1;
    }
    mult = am;
    plus = ap;
}

__device__ __forceinline__ uint64_t pcg_out(U128 s) {
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = unsigned(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct DrawParams {
    const uint64_t *rng;  // [chains][4] state lo, hi, inc lo, hi
    const uint32_t *buf;  // [chains][2] has_uint32, cached
    int V, n_dev, budget;
    uint64_t lim;         // hit iff word < lim (all_hit: every word)
    int all_hit;
    int32_t *moff;        // [chains][budget + 1], absolute into mpos / mval
    int32_t *mpos;        // [chains * cap]
    uint8_t *mval;
    int64_t cap;
    int32_t *status;      // [chains] 0 ok, 1 list overflow, 2 rejection
};

__global__ void __launch_bounds__(kT) ea_draw_kernel(const DrawParams d) {
    const int c = blockIdx.x, t = threadIdx.x;
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t *hit_idx = reinterpret_cast<uint64_t *>(sm);       // [kT * kW]
    uint64_t *hit_nxt = hit_idx + kT * kW;                       // [kT * kW]
    __shared__ int s_cnt[kT];
    __shared__ int s_done, s_total;
    const U128 inc{d.rng[4 * c + 2], d.rng[4 * c + 3]};
    U128 bs{d.rng[4 * c], d.rng[4 * c + 1]};  // state before the block's first word
    U128 tm, tp, bm, bp;
    lcg_jump(uint64_t(t) * kW, inc, tm, tp);
    lcg_jump(uint64_t(kT) * kW, inc, bm, bp);
    // walker state (thread 0)
    uint64_t wp = 0;  // next word index to be consumed as random()
    int64_t child = 0, pos = 0, nmut = 0;
    uint32_t has = d.buf[2 * c], cached = d.buf[2 * c + 1];
    const int64_t base = int64_t(c) * d.cap;
    int32_t *moff = d.moff + int64_t(c) * (d.budget + 1);
    int st = 0;
    if (t == 0) {
        moff[0] = int32_t(base);
        s_done = d.budget <= 0;
    }
    __syncthreads();
    uint64_t block = 0;
    // advance (child, pos) over n random() misses, closing finished children
    auto advance = [&](uint64_t n) {
        int64_t total = pos + int64_t(n);
        while (total >= d.V && child < d.budget) {
            total -= d.V;
            ++child;
            moff[child] = int32_t(base + nmut);
        }
        pos = child < d.budget ? total : 0;
    };
    while (!s_done) {
        // parallel phase: this thread's W words (+1 peeked)
        U128 s = add128(mul128(tm, bs), tp);
        uint64_t w[kW + 1];
#pragma unroll
        for (int k = 0; k <= kW; ++k) {
            s = add128(mul128(s, pcg_mult()), inc);
            w[k] = pcg_out(s);
        }
        int n = 0;
#pragma unroll
        for (int k = 0; k < kW; ++k) n += (d.all_hit || w[k] < d.lim) ? 1 : 0;
        s_cnt[t] = n;
        __syncthreads();
        if (t == 0) {  // exclusive scan (one thread: 256 adds)
            int acc = 0;
            for (int q = 0; q < kT; ++q) {
                const int v = s_cnt[q];
                s_cnt[q] = acc;
                acc += v;
            }
        }
        __syncthreads();
        int o = s_cnt[t];
        const uint64_t first = block + uint64_t(t) * kW;
#pragma unroll
        for (int k = 0; k < kW; ++k)
            if (d.all_hit || w[k] < d.lim) {
                hit_idx[o] = first + k;
                hit_nxt[o] = w[k + 1];
                ++o;
            }
        if (t == kT - 1) s_total = o;  // last offset + its count
        __syncthreads();
        if (t == 0) {
            const int nh = s_total;
            const uint64_t end = block + uint64_t(kT) * kW;
            for (int q = 0; q < nh && child < d.budget && !st; ++q) {
                const uint64_t h = hit_idx[q];
                if (h < wp) continue;  // consumed by an integers() draw
                advance(h - wp);
                if (child >= d.budget) break;
                // rng.integers(n_dev): Lemire on a buffered 32-bit draw
                uint32_t val = 0;
                wp = h + 1;
                if (d.n_dev > 1) {
                    uint32_t x;
                    if (has) {
                        x = cached;
                        has = 0;
                    } else {
                        const uint64_t nx = hit_nxt[q];
                        x = uint32_t(nx);
                        cached = uint32_t(nx >> 32);
                        has = 1;
                        wp = h + 2;
                    }
                    const uint64_t m = uint64_t(x) * uint32_t(d.n_dev);
                    const uint32_t left = uint32_t(m);
                    if (left < uint32_t(d.n_dev)) {
                        const uint32_t thr =
                            (0xFFFFFFFFu - uint32_t(d.n_dev - 1)) % uint32_t(d.n_dev);
                        if (left < thr) {
                            st = 2;  // rejection: the host redraws this chain
                            break;
                        }
                    }
                    val = uint32_t(m >> 32);
                }
                if (nmut >= d.cap) {
                    st = 1;
                    break;
                }
                d.mpos[base + nmut] = int32_t(pos);
                d.mval[base + nmut] = uint8_t(val);
                ++nmut;
                advance(1);
            }
            if (!st && child < d.budget && wp < end) {
                advance(end - wp);
                wp = end;
            }
            s_done = st || child >= d.budget;
        }
        __syncthreads();
        block += uint64_t(kT) * kW;
        bs = add128(mul128(bm, bs), bp);
    }
    if (t == 0) {
        // (also after a failure: the lists stay well formed, truncated)
        for (int64_t k = child + 1; k <= d.budget; ++k) moff[k] = int32_t(base + nmut);
        d.status[c] = st;
    }
}

}  // namespace

extern "C" int hs_ea_draw(int32_t chains, const uint64_t *d_rng, const uint32_t *d_buf,
                          int32_t n_tasks, int32_t n_dev, double p, int32_t budget,
                          int32_t *d_moff, int32_t *d_mpos, uint8_t *d_mval,
                          int64_t cap_per_chain, int32_t *d_status, void *stream) {
    if (chains < 1 || !d_rng || !d_buf || n_tasks < 1 || n_dev < 1 || n_dev > 256 ||
        budget < 0 || !d_moff || !d_status || cap_per_chain < 1 || !d_mpos || !d_mval ||
        !(p >= 0.0))
        return hs::set_error(HS_EINVAL, "hs_ea_draw: bad arguments");
    DrawParams d{};
    d.rng = d_rng;
    d.buf = d_buf;
    d.V = n_tasks;
    d.n_dev = n_dev;
    d.budget = budget;
    // random() < p  <=>  (w >> 11) < ceil(p * 2^53)  <=>  w < ceil(p * 2^53) << 11
    const double t53 = std::ceil(p * 9007199254740992.0);
    if (t53 >= 9007199254740992.0) {
        d.all_hit = 1;
        d.lim = 0;
    } else {
        d.lim = uint64_t(t53) << 11;
    }
    d.moff = d_moff;
    d.mpos = d_mpos;
    d.mval = d_mval;
    d.cap = cap_per_chain;
    d.status = d_status;
    const size_t smem = size_t(kT) * kW * 16;
    cudaError_t e = cudaFuncSetAttribute(ea_draw_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e == cudaSuccess) {
        ea_draw_kernel<<<chains, kT, smem, static_cast<cudaStream_t>(stream)>>>(d);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess)
        return hs::set_error(HS_ECUDA, std::string("hs_ea_draw: ") + cudaGetErrorString(e));
    return HS_OK;
}
