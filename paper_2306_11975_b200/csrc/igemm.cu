// igemm.cu -- A4 + A5 of the Ozaki scheme on sm_100a in ONE persistent kernel:
//   INT8 x INT8 -> INT32 slice-pair GEMMs on tcgen05 tensor cores (Alg. 3 line 6)
//   + the FP64 accumulation / scaling epilogue (Alg. 3 line 7),
// replacing the paper's cublasGemmEx-per-pair + separate FP64 accumulation kernel
// (whose accumulation pass was HBM-bound at ~90% of DRAM BW).
//
// Design:
//  * Output tile = 128 rows x NC columns of C, one CTA per SM (persistent, grouped raster,
//    soft per-wave grid barrier so CTAs sharing operands stream K through L2 together, odd
//    waves walking K backwards), CTAs in clusters of two sharing A tiles by TMA multicast.
//  * Warp roles: 4 epilogue warps, 1 TMA producer, 2 MMA issuers taking alternate A-slice
//    tiles (one issuer leaves the tensor pipe idle during its per-tile barrier wait).
//  * K is processed in k-blocks of 128 bytes (one 128B-swizzle row).  Per k-block ONE 3-D
//    TMA box brings all s B-slice tiles of the NC columns (B planes are stored in reversed
//    slice order q -> s-q) into the B ring, and the s A-slice tiles (128 x 128 B each) flow
//    one by one through a deeper A ring.
//  * Operand sharing: for A-slice p, its partners B^(1..s+1-p) are the contiguous
//    "window" of reversed B blocks [p-1, s-1]; tcgen05.mma instructions with
//    N = (s+1-p) NC (split into <= 256-wide pieces) multiply A^(p) by the whole window,
//    and window block j lands in TMEM column block j, which always holds level g = s+1-j.
//    So TMEM accumulates the exact per-level sums L_g directly: each A and B slice tile
//    is loaded once per k-block and every pair i+j <= s+1 is covered.
//  * INT32 budget: a level has <= s pairs; when s * k * (2^w-1)^2 > 2^31-1 the
//    pairs of the top levels go to a second TMEM region (T = 2), else K is processed in
//    chunks and between chunks the epilogue drains TMEM into exact int64 partial sums
//    (per-CTA global scratch).  MMAs only accumulate: the epilogue zeroes what it read.
//  * Epilogue (4 warps, TMEM lane quarter = warp % 4): L_g -> FP64 in the canonical
//    order g = s+1 .. 2 (reading A6), ldexp by E_A+E_B (A7), alpha/beta (A8), NaN rows (A9),
//    coalesced column-major stores of C.
#include <cstdlib>

#include "igemm_kernel.cuh"

namespace ozimmu {
using namespace gemm_detail;

namespace gemm_detail {
#define OZ_EXTERN(S) extern template cudaError_t launch_t<S>(const GemmArgs &, const GemmPlan &, \
                                                             EpiMode, cudaStream_t);
OZ_EXTERN(1) OZ_EXTERN(2) OZ_EXTERN(3) OZ_EXTERN(4) OZ_EXTERN(5) OZ_EXTERN(6) OZ_EXTERN(7)
OZ_EXTERN(8) OZ_EXTERN(9) OZ_EXTERN(10) OZ_EXTERN(11) OZ_EXTERN(12) OZ_EXTERN(13) OZ_EXTERN(14)
OZ_EXTERN(15) OZ_EXTERN(16) OZ_EXTERN(17) OZ_EXTERN(18) OZ_EXTERN(19) OZ_EXTERN(20)
OZ_EXTERN(21) OZ_EXTERN(22) OZ_EXTERN(23) OZ_EXTERN(24) OZ_EXTERN(25) OZ_EXTERN(26)
OZ_EXTERN(27) OZ_EXTERN(28) OZ_EXTERN(29) OZ_EXTERN(30) OZ_EXTERN(31) OZ_EXTERN(32)
#undef OZ_EXTERN
#define OZ_EXTERN32(S) extern template cudaError_t launch_t<S, 32>(const GemmArgs &, \
                                                                const GemmPlan &, EpiMode, \
                                                                cudaStream_t);
OZ_EXTERN32(1) OZ_EXTERN32(2) OZ_EXTERN32(3) OZ_EXTERN32(4) OZ_EXTERN32(5) OZ_EXTERN32(6)
OZ_EXTERN32(7) OZ_EXTERN32(8) OZ_EXTERN32(9) OZ_EXTERN32(10)
#undef OZ_EXTERN32
}  // namespace gemm_detail

// INT32 budget of one accumulator region over the whole K: no K chunks needed
// when a level's pairs fit one region, or two regions of G pairs (T = 2) fit TMEM.
static bool budget_one_chunk(int s, int w, int64_t k_pad, int nc) {
    const int64_t d = ((int64_t)1 << w) - 1;
    const int64_t kfull = ceil_div(k_pad, kKB) * kKB;
    const int64_t G = (int64_t)2147483647 / (kfull * d * d);
    if (G >= s) return true;
    return G >= 1 && (s + G - 1) / G == 2 && ((int64_t)s + (s - G)) * nc <= 512;
}

int sk_mode() {
    static const int m = getenv("OZIMMU_SK") ? atoi(getenv("OZIMMU_SK")) : 0;
    return m;
}

bool plan_gemm(int s, int w, int64_t m, int64_t n, int64_t k_pad, int num_sms, GemmPlan *p) {
    if (s < 1 || s > 32 || w < 1) return false;
    int nc = nc_for(s);
    // Stream-K (OZIMMU_SK: 0 off = default, 1 forced, -1 auto): when the tiles of a problem fill
    // only a few waves and the last one is partial, clusters share the K loop of the tail
    // units instead (k_oz_gemm); then the default tile width keeps its better MMA mix.  Needs
    // one INT32-safe pass over K (no K chunks).  Off by default: measured slower than the
    // data-parallel schedule at 1024^3-2048^3 (53 -> 90 us and 261 -> 313 us GEMM), the
    // fixup's L2 round trips for a split unit's int32 partials (s N_c values per row) cost
    // more than the partial wave they remove.  Bit-identical either way.
    const int sk_env = sk_mode();
    bool sk = false;
    if (sk_env != 0 && budget_one_chunk(s, w, k_pad, nc)) {
        const int64_t units = ceil_div(m, kBlockM) * ceil_div(ceil_div(n, (int64_t)nc), 2);
        const int64_t G = num_sms / 2 > 0 ? num_sms / 2 : 1;  // CTA pairs
        const int64_t waves = ceil_div(units, G);
        // partial last wave costing > 2 % of a data-parallel schedule of <= 8 waves
        sk = sk_env == 1 || (waves <= 8 && (waves * G - units) * 50 > waves * G);
    }
    // Small problems without stream-K: with few tiles the last, partial wave dominates; N_c =
    // 32 gives 1.5-2x the tiles (an instance exists for s <= 10) at ~4 % lower MMA-mix
    // efficiency.  Measured crossover: better up to ~5 waves of default tiles (1024^3 GEMM
    // 67 -> 47 us).
    if (!sk && nc > 32 && s <= 10 &&
        ceil_div(m, kBlockM) * ceil_div(n, (int64_t)nc) <= 5 * (int64_t)num_sms)
        nc = 32;
    // Short K: a tile's MMAs take only ~num_kb x the epilogue's TMEM drain, which a single
    // accumulator leaves exposed; two accumulator buffers (2 s N_c <= 512 TMEM columns) let
    // the next tile's MMAs run during the drain.  For s <= 8 the N_c = 32 instance fits two.
    const int64_t num_kb0 = ceil_div(k_pad, kKB);
    static const int acc2_env = getenv("OZIMMU_ACC2") ? atoi(getenv("OZIMMU_ACC2")) : -1;
    bool acc2 = false;
    if (!sk && acc2_env != 0) {
        if (2 * s * nc <= 512) acc2 = true;
        // measured: d = 8 quantum gate (K' = 512, 4 k-blocks) GEMM 13.0 -> 11.7 ms; at 16
        // k-blocks the narrower tile's MMA mix costs more than the drain (28.6 -> 29.6 ms)
        else if (s <= 8 && (num_kb0 <= 8 || acc2_env == 1)) { nc = 32; acc2 = true; }
    }
    const size_t smem_budget = 232448 - 3072;  // 227 KB opt-in max minus barriers/align/static
    const size_t b_stage = (size_t)s * nc * kKB;
    const size_t a_stage = (size_t)kBlockM * kKB;
    static const char *bs_env = getenv("OZIMMU_B_STAGES");  // experiments
    static const char *as_env = getenv("OZIMMU_A_STAGES");
    const int b_stages = bs_env ? atoi(bs_env) : 2;
    if (b_stages * b_stage + 2 * a_stage > smem_budget) return false;
    int a_stages = (int)((smem_budget - b_stages * b_stage) / a_stage);
    if (a_stages > 12) a_stages = 12;
    if (as_env && atoi(as_env) >= 2 && atoi(as_env) < a_stages) a_stages = atoi(as_env);
    // even: the two MMA issuer warps take alternate A tiles, so with an even ring every slot
    // always belongs to the same warp (k_oz_gemm's parity waits rely on it)
    a_stages &= ~1;
    if (a_stages < 2) return false;
    // INT32 budget: an accumulator holding `g` pair products over K' values of k
    // needs g * K' * (2^w - 1)^2 <= 2^31 - 1.  Level g = s+1 has s pairs.  Prefer splitting the
    // pairs of a level over T = 2 TMEM regions (sub-groups of G pairs) over draining K chunks.
    const int64_t d = ((int64_t)1 << w) - 1;
    const int64_t num_kb = ceil_div(k_pad, kKB);
    const int64_t kfull = num_kb * kKB;
    const int64_t G = (int64_t)2147483647 / (kfull * d * d);
    p->T = 1;
    p->G = s;
    p->chunk_blocks = num_kb;
    if (G < s) {
        const int64_t blocks2 = (int64_t)s + (s - G);
        if (G >= 1 && (s + G - 1) / G == 2 && blocks2 * nc <= 512) {
            p->T = 2;
            p->G = (int)G;
        } else {
            const int64_t kmax = (int64_t)2147483647 / ((int64_t)s * d * d);
            p->chunk_blocks = kmax / kKB;
            if (p->chunk_blocks < 1) return false;
        }
    }
    if (p->T == 2 || p->chunk_blocks < num_kb) acc2 = false;  // one INT32-safe period per tile
    p->nacc = acc2 ? 2 : 1;
    p->tile_n = nc;
    p->k_block = kKB;
    p->a_stages = a_stages;
    p->b_stages = b_stages;
    p->stages = a_stages;
    p->num_k_blocks = num_kb;
    p->k_chunks = (int)ceil_div(p->num_k_blocks, p->chunk_blocks);
    if (p->k_chunks < 1) p->k_chunks = 1;
    const int64_t tiles = ceil_div(m, kBlockM) * ceil_div(n, nc);
    p->grid = (int)(tiles < num_sms ? tiles : num_sms);
    if (p->grid < 1) p->grid = 1;
    // stream-K counter slots: units x cluster size <= (tiles_m + 1) x (tiles_n + 1)
    p->tiles = (ceil_div(m, kBlockM) + 1) * (ceil_div(n, nc) + 1);
    p->sk = sk && p->k_chunks == 1 ? 1 : 0;
    if (p->sk) {
        // every cluster takes a share of the K loops, but a unit is cut into at most ~4 parts
        // (fewer for short K: each part's partial sums cost a write and a read in the fixup)
        int64_t parts = p->num_k_blocks / 4;
        parts = parts < 1 ? 1 : (parts > 4 ? 4 : parts);
        const int64_t g = tiles * parts;
        p->grid = (int)(g < num_sms ? g : num_sms);
    }
    p->smem_bytes = 1024 /*align slack*/ + b_stage * b_stages + a_stage * a_stages +
                    8 * (2 * b_stages + 2 * a_stages + 4) + 16;
    int cols = 32;
    const int used = (p->T == 2 ? 2 * s - p->G : s) * nc;
    while (cols < used) cols <<= 1;
    if (p->nacc == 2) cols *= 2;  // buffer 1 at column cols / 2
    p->tmem_cols = cols;
    return true;
}

// Stream-K scratch: arrival counters [units x cl <= tiles + 4] then int32 partial level sums
// [grid CTAs][2 slots][used TMEM columns <= 512][128 rows].
static size_t sk_scratch(int64_t tiles, int grid) {
    const size_t cnt = ((size_t)(tiles + 4) * sizeof(int) + 255) / 256 * 256;
    return cnt + (size_t)grid * 2 * 512 * kBlockM * sizeof(int32_t);
}
size_t sk_counters_bytes(int64_t tiles) { return ((size_t)(tiles + 4) * sizeof(int) + 255) / 256 * 256; }

size_t chunk_scratch_bytes(const GemmPlan &p, int s) {
    if (p.sk) return sk_scratch(p.tiles, p.grid);
    if (p.k_chunks <= 1) return 0;
    return (size_t)p.grid * s * p.tile_n * kBlockM * sizeof(int64_t);
}

// Upper bound of chunk_scratch_bytes over every SM cap (ozimmu_set_max_sms) and device of up to
// max_sms SMs: the tile width may switch between 32 and nc_for(s) with the cap (small-problem
// rule in plan_gemm), and the grid is at most max_sms CTAs.
size_t chunk_scratch_bound(const GemmPlan &p, int s, int max_sms) {
    const int g = p.grid > max_sms ? p.grid : max_sms;
    // stream-K may be chosen under any SM cap / for any sub-shape with one pass over K; its
    // counters are bounded by the tiles of the narrowest tile width
    const size_t skb = sk_mode() != 0 ? sk_scratch(p.tiles * (p.tile_n / 16 > 0 ? p.tile_n / 16 : 1), g)
                                      : 0;
    const int nc = nc_for(s) > p.tile_n ? nc_for(s) : p.tile_n;
    // K chunks in this plan, or possibly under an SM cap: two INT32 regions that fit TMEM only
    // thanks to the narrow small-problem tile may not fit with the default width
    const bool chunks = p.k_chunks > 1 || (p.T == 2 && p.tile_n < nc_for(s));
    const size_t kcb = chunks ? (size_t)g * s * nc * kBlockM * sizeof(int64_t) : 0;
    return skb > kcb ? skb : kcb;
}

cudaError_t launch_gemm(const GemmArgs &a, const GemmPlan &p, EpiMode mode, cudaStream_t st,
                        int *launches) {
    if (a.m <= 0 || a.n <= 0) return cudaSuccess;
    cudaError_t e;
    if (p.tile_n == 32 && nc_for(a.s) != 32) {  // small-problem instances (s <= 10)
        switch (a.s) {
#define OZ_CASE32(S) case S: e = launch_t<S, 32>(a, p, mode, st); break;
        OZ_CASE32(1) OZ_CASE32(2) OZ_CASE32(3) OZ_CASE32(4) OZ_CASE32(5) OZ_CASE32(6)
        OZ_CASE32(7) OZ_CASE32(8) OZ_CASE32(9) OZ_CASE32(10)
#undef OZ_CASE32
        default: return cudaErrorInvalidValue;
        }
        ++*launches;
        return e;
    }
    switch (a.s) {
#define OZ_CASE(S) case S: e = launch_t<S>(a, p, mode, st); break;
    OZ_CASE(1) OZ_CASE(2) OZ_CASE(3) OZ_CASE(4) OZ_CASE(5) OZ_CASE(6) OZ_CASE(7) OZ_CASE(8)
    OZ_CASE(9) OZ_CASE(10) OZ_CASE(11) OZ_CASE(12) OZ_CASE(13) OZ_CASE(14) OZ_CASE(15)
    OZ_CASE(16) OZ_CASE(17) OZ_CASE(18) OZ_CASE(19) OZ_CASE(20) OZ_CASE(21) OZ_CASE(22)
    OZ_CASE(23) OZ_CASE(24) OZ_CASE(25) OZ_CASE(26) OZ_CASE(27) OZ_CASE(28) OZ_CASE(29)
    OZ_CASE(30) OZ_CASE(31) OZ_CASE(32)
#undef OZ_CASE
    default: return cudaErrorInvalidValue;
    }
    ++*launches;
    return e;
}

}  // namespace ozimmu
