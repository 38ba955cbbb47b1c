// Onesweep LSD radix sort of the key-sort binning path (shuffled input):
// linear cell ids (32-bit keys) with their input indices, 8-bit digits, one launch per pass.
//
// The digit histograms of every pass come from k_lkey (one read of the keys for all passes).
// Within a pass, tiles of OS_TILE keys are taken in order from an atomic counter; each tile
// ranks its keys by digit in shared memory, publishes its per-digit counts, and finds its
// per-digit output offsets by a decoupled look-back over the earlier tiles' published state
// (an aggregate, or an inclusive prefix that ends the look-back).  The tile is then written
// digit run by digit run (coalesced).  Stable: within a digit, tiles are in order and keys
// inside a tile keep their order (warp, iteration, lane).
//
// Look-back state: two arrays of tiles x 256 words, used by alternate passes; a word is 0 (not
// published), count + 1 (aggregate) or OS_PREFIX | inclusive prefix.  k_lkey zeroes the
// first; pass p zeroes its own rows of the other one for pass p + 1.
#include "fec_kernels.cuh"

namespace fec {

constexpr int OS_THREADS = 256, OS_ITEMS = 16, OS_TILE = OS_THREADS * OS_ITEMS;
constexpr uint32_t OS_PREFIX = 0x80000000u;
// 3 resident blocks per SM (registers <= 85): the look-back and the digit-run stores of
// one tile overlap the loads and ranking of the others (2 blocks: 1.4 TB/s per pass on C5)
constexpr int OS_MIN_BLOCKS = 3;
static_assert(OS_TILE == RS_TILE, "onesweep tiles = radix tiles (workspace sizing)");

__device__ __forceinline__ uint32_t ld_state(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_state(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(OS_THREADS, OS_MIN_BLOCKS) k_onesweep(const Grid* __restrict__ gp, int pass, uint32_t* __restrict__ k0,
                                                        int* __restrict__ v0, uint32_t* __restrict__ k1,
                                                        int* __restrict__ v1, int64_t n,
                                                        const uint32_t* __restrict__ ghist,
                                                        uint32_t* __restrict__ state, int64_t tiles,
                                                        unsigned int* __restrict__ tile_ctr) {
    pdl_prologue();
    if (gp->status || !gp->key_sort || pass >= gp->passes) return;
    const uint32_t* __restrict__ kin = (pass & 1) ? k1 : k0;
    const int* __restrict__ vin = (pass & 1) ? v1 : v0;
    uint32_t* __restrict__ kout = (pass & 1) ? k0 : k1;
    int* __restrict__ vout = (pass & 1) ? v0 : v1;
    uint32_t* cur = state + (int64_t)(pass & 1) * tiles * 256;
    uint32_t* nxt = state + (int64_t)((pass + 1) & 1) * tiles * 256;
    const int shift = 8 * pass;

    __shared__ uint32_t wcnt[OS_THREADS / kWarp][256];
    __shared__ uint32_t gofs[256];
    __shared__ uint32_t tstart[256];
    __shared__ uint32_t sk[OS_TILE];
    __shared__ int sv[OS_TILE];
    __shared__ unsigned int tile_sh;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    // persistent blocks: tiles in counter order (a tile only waits on earlier tiles, which
    // blocks already running hold)
    while (true) {
    __syncthreads();
    if (tid == 0) tile_sh = atomicAdd(tile_ctr + pass, 1u);
    for (int d = tid; d < (OS_THREADS / kWarp) * 256; d += OS_THREADS) (&wcnt[0][0])[d] = 0u;
    __syncthreads();
    const unsigned tile = tile_sh;
    if ((int64_t)tile >= tiles) return;
    const int64_t tbase = (int64_t)tile * OS_TILE;
    const int64_t base = tbase + (int64_t)w * (OS_ITEMS * kWarp);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t k[OS_ITEMS];
    int v[OS_ITEMS];
    uint32_t rank[OS_ITEMS];
    const int64_t nvalid = n - base;  // items it with it * kWarp + lane < nvalid are keys
#pragma unroll
    for (int it = 0; it < OS_ITEMS; ++it) {
        const int64_t i = base + it * kWarp + lane;
        const bool ok = i < n;
        k[it] = ok ? __ldg(kin + i) : 0u;
        v[it] = ok ? __ldg(vin + i) : 0;
    }
    // rank inside the warp's 512 keys (iteration-major, lane-minor = input order)
#pragma unroll
    for (int it = 0; it < OS_ITEMS; ++it) {
        const int d = (it * kWarp + lane < nvalid) ? (int)((k[it] >> shift) & 255u) : 256;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t c = d < 256 ? wcnt[w][d] : 0u;
        __syncwarp();
        rank[it] = c + __popc(peers & lt);
        if (d < 256 && (peers & lt) == 0u) wcnt[w][d] = c + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit (thread d): exclusive offsets of the warps, the tile's count
    const int d = tid;
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < OS_THREADS / kWarp; ++ww) {
        const uint32_t t = wcnt[ww][d];
        wcnt[ww][d] = cnt;
        cnt += t;
    }
    tstart[d] = cnt;
    // publish, then look back over earlier tiles for this digit
    uint32_t excl = 0;
    if (tile == 0) {
        st_state(cur + d, OS_PREFIX | cnt);
    } else {
        st_state(cur + (int64_t)tile * 256 + d, cnt + 1u);
        int64_t j = (int64_t)tile - 1;
        while (true) {
            const uint32_t s = ld_state(cur + j * 256 + d);
            if (s == 0u) continue;
            if (s & OS_PREFIX) {
                excl += s & ~OS_PREFIX;
                break;
            }
            excl += s - 1u;
            --j;
        }
        st_state(cur + (int64_t)tile * 256 + d, OS_PREFIX | (excl + cnt));
    }
    nxt[(int64_t)tile * 256 + d] = 0u;  // the next pass's state row (that array's last user is done)
    __syncthreads();
    // exclusive scans over the 256 digits (warp 0): tile-local starts and global digit starts
    if (w == 0) {
        uint32_t a[8], b[8], sa = 0, sb = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            a[j] = tstart[8 * lane + j];
            b[j] = __ldg(ghist + pass * 256 + 8 * lane + j);
            sa += a[j];
            sb += b[j];
        }
        uint32_t xa = sa, xb = sb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, o);
            const uint32_t yb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= o) {
                xa += ya;
                xb += yb;
            }
        }
        uint32_t ra = xa - sa, rb = xb - sb;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            tstart[8 * lane + j] = ra;
            gofs[8 * lane + j] = rb;  // global start of the digit
            ra += a[j];
            rb += b[j];
        }
    }
    __syncthreads();
    gofs[d] += excl;  // + the digit's keys in earlier tiles
    // stage the tile in digit order
#pragma unroll
    for (int it = 0; it < OS_ITEMS; ++it) {
        const int dd = (it * kWarp + lane < nvalid) ? (int)((k[it] >> shift) & 255u) : 256;
        if (dd < 256) {
            const uint32_t lp = tstart[dd] + wcnt[w][dd] + rank[it];
            sk[lp] = k[it];
            sv[lp] = v[it];
        }
    }
    __syncthreads();
    const int cntt = (int)min((int64_t)OS_TILE, n - tbase);
    for (int lp = tid; lp < cntt; lp += OS_THREADS) {
        const uint32_t key = sk[lp];
        const int dd = (int)((key >> shift) & 255u);
        const uint32_t pos = gofs[dd] + ((uint32_t)lp - tstart[dd]);
        kout[pos] = key;
        vout[pos] = sv[lp];
    }
    }  // tiles
}

}  // namespace fec
