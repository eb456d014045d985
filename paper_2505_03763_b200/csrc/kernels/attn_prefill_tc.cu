// Prefill attention on the 5th-generation tensor cores (sm_100a tcgen05/TMEM).
//
// Causal flash attention for a varlen batch of prompts over the paged KV cache
// (GQA).  One CTA = 128 query rows of one prompt for TWO query heads of the
// same kv head: two independent 128-thread groups (warps 0-3 | 4-7), each with
// its own S/O accumulators in TMEM, P buffer, MMA-issuing thread and barriers,
// sharing the K/V blocks -- while one group runs its softmax the tensor core
// works on the other group's MMAs.  Thread t of a group owns query row t (TMEM
// lane t).  Per 128-key block j and group:
//   S  = Q K_j^T        tcgen05.mma M=128 N=128 K=hd, Q and K from smem
//                       (TMA SWIZZLE_128B, K-major), S fp32 in TMEM cols [0,128)
//   softmax             each thread tcgen05.ld's its S row twice (max, then
//                       exp2/sum), online max/sum in fp32 (log2 domain), P as
//                       fp16 into smem in the K-major 128B-swizzled layout
//   O += P V_j          tcgen05.mma M=128 N=hd K=128, P (K-major) and V from
//                       smem -- V is [keys][hd] as stored, i.e. MN-major for
//                       the B operand (instruction-descriptor transpose bit);
//                       O fp32 in TMEM cols [128, 128+hd), rescaled in place
//                       (tcgen05.ld/st) only when a row's max moved.
// Q (a 3-D TMA map over [tokens][H][hd]) and K/V (one 16-row TMA box per page
// slice, the arena-wide map of the decode attention) are loaded by thread 0:
// K double-buffered (block j+1 lands while block j's softmax runs), V single
// (block j+1's V lands during the next S MMA and softmax); a stage is reloaded
// once both groups' MMAs released it (count-2 "empty" barriers).  smem: 144 KB
// (hd 64) / 224 KB (hd 128), TMEM: 512 columns -- one CTA per SM.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "attention.cuh"
#include "common.cuh"

namespace sw {
int stream_sm_count(cudaStream_t st);  // engine/partition.cu

namespace {

constexpr int kRows = 128;     // query rows per CTA
constexpr int kBlk = 128;      // keys per block
constexpr int kPg = 16;        // tokens per page

__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 3-D TMA load (inner, middle, outer coordinates).
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_addr(dst)),
        "l"(tmap), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// 32 lanes x 32 fp32 columns, registers -> TMEM (inverse of tmem_ld32).
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// B operand stored MN-major (N contiguous) in 128B-swizzled atoms of 64 N x
// 8 K rows: SBO = 1024 B between 8-row K groups, LBO = distance between
// 64-wide N groups.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_byte_addr, uint32_t lbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_byte_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

template <int HD>
struct TcCfg {
    static constexpr int NH = HD / 64;                 // 64-wide column atoms of a head row
    static constexpr int kAtom = kRows * 128;          // one [128 rows][128 B] atom column
    static constexpr int kQ = NH * kAtom;              // one group's Q tile
    static constexpr int kKV = NH * kAtom;             // one K (or V) block of 128 keys
    static constexpr int kP = 2 * kAtom;               // P: 128 rows x 128 keys bf16
    static constexpr int kOffK = 2 * kQ;               // K: two stages
    static constexpr int kOffV = kOffK + 2 * kKV;      // V: one stage
    static constexpr int kOffP = kOffV + kKV;          // P: one per group
    static constexpr int kOffBar = kOffP + 2 * kP;
    static constexpr int kSmem = 1024 + kOffBar + 128;
    static_assert(kSmem <= 227 * 1024, "smem budget");
    static constexpr uint32_t kTmemCols = 512;          // group g: S [256g, 256g+128), O [256g+128, +HD)
};

template <int HD>
__global__ void __launch_bounds__(256, 1) attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                              const __grid_constant__ CUtensorMap tm_kv,
                                                              __nv_bfloat16* __restrict__ out, PrefillTcArgs a) {
    using C = TcCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + C::kOffK;
    uint8_t* sV = smem + C::kOffV;
    uint8_t* sP = smem + C::kOffP;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* q_full = bar;
    uint64_t* k_full = bar + 1;   // [2]
    uint64_t* k_empty = bar + 3;  // [2] both groups' S MMAs of the stage retired
    uint64_t* v_full = bar + 5;
    uint64_t* v_empty = bar + 6;  // both groups' PV MMAs retired
    uint64_t* s_done_g = bar + 7;  // [2] per group
    uint64_t* o_done_g = bar + 9;  // [2] per group
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 11);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int g = warp >> 2;              // group: query head 2 * pair + g
    const int gt = tid & 127;             // thread within the group = query row
    if (tid == 0) {
        mbar_init(q_full, 1);
        mbar_init(&k_full[0], 1);
        mbar_init(&k_full[1], 1);
        mbar_init(&k_empty[0], 2);
        mbar_init(&k_empty[1], 2);
        mbar_init(v_full, 1);
        mbar_init(v_empty, 2);
        for (int q = 0; q < 2; ++q) {
            mbar_init(&s_done_g[q], 1);
            mbar_init(&o_done_g[q], 1);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_kv);
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem + 256 * g, tO = tS + kBlk;
    uint64_t* s_done = &s_done_g[g];
    uint64_t* o_done = &o_done_g[g];
    uint8_t* sQg = sQ + g * C::kQ;
    uint8_t* sPg = sP + g * C::kP;

    // Persistent: work items (128-row query tile, head pair) dealt to the CTAs last tile first
    // (a prompt's later query tiles attend to more keys) in a snake order -- round k runs
    // left to right when k is even, right to left when odd -- so the heavy and light items
    // of consecutive rounds pair up on one CTA.  With one CTA per item (non-persistent) the
    // same mapping makes the hardware's in-order block issue longest-first (8B 4 x 8192:
    // 4.36 -> 4.26 ms per layer).  Barrier phases run on the CTA's global key-block count
    // gb (K stage gb & 1) and item count it.
    const int pairs = a.H / 2;
    const int n_items = *a.n_tiles * pairs;
    const int G = static_cast<int>(gridDim.x), bx = static_cast<int>(blockIdx.x);
    int gb = 0, it = 0;
    for (int k = 0;; ++k, ++it) {
    const int idx = k * G + ((k & 1) ? G - 1 - bx : bx);
    if (idx >= n_items) break;
    const int item = n_items - 1 - idx;
    const int tile = item / pairs, pair = item % pairs;
    const int h = 2 * pair + g;
    const int hk = h / (a.H / a.Hkv);     // same for both groups (H / Hkv even)
    const int sq = a.tile_seq[tile];
    const int q0 = a.tile_q0[tile];
    const int start = a.cu_seqlens[sq];
    const int len = a.cu_seqlens[sq + 1] - start;
    const int kend = min(q0 + kRows, len);        // keys this tile attends to: [0, kend)
    const int nblk = (kend + kBlk - 1) / kBlk;
    const int npages = (len + kPg - 1) / kPg;
    const int32_t* ptab = a.page_table + static_cast<long long>(a.seq_slot[sq]) * a.max_pages;

    // K (v = 0) or V (v = 1) of key block j into `dst`, completing on `b` (thread 0).
    // Page ids past the prompt read page 0 (finite data, masked).
    auto load_blk = [&](int j, int v, uint8_t* dst, uint64_t* b) {
        const uint64_t pol = l2_policy_evict_last();  // re-read by the prompt's later query tiles
        int pid[kBlk / kPg];
#pragma unroll
        for (int i = 0; i < kBlk / kPg; ++i) {
            const int pg = j * (kBlk / kPg) + i;
            pid[i] = pg < npages ? ptab[pg] : 0;
        }
        mbar_expect_tx(b, C::kKV);
#pragma unroll
        for (int i = 0; i < kBlk / kPg; ++i) {
            const int kr = a.layer_row0 + pid[i] * a.page_rows + hk * kPg + (v ? a.v_rows : 0);
#pragma unroll
            for (int c = 0; c < C::NH; ++c) tma_load_2d(dst + c * C::kAtom + i * kPg * 128, &tm_kv, b, c * 64, kr, pol);
        }
    };
    if (tid == 0) {
        // the previous item's S MMAs (both groups) retired: Q and that K stage are free
        if (gb >= 1) mbar_wait(&k_empty[(gb - 1) & 1], ((gb - 1) >> 1) & 1);
        mbar_expect_tx(q_full, 2 * C::kQ);
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int c = 0; c < C::NH; ++c)
                tma_load_3d(sQ + q * C::kQ + c * C::kAtom, &tm_q, q_full, c * 64, 2 * pair + q, start + q0);
        if (gb >= 2) mbar_wait(&k_empty[gb & 1], ((gb - 2) >> 1) & 1);
        load_blk(0, 0, sK + (gb & 1) * C::kKV, &k_full[gb & 1]);
        if (gb >= 1) mbar_wait(v_empty, (gb - 1) & 1);  // both groups' last PV retired: V is free
        load_blk(0, 1, sV, v_full);
    }

    // fp16 operands (q, K/V cache, P: common.cuh kv_t)
    constexpr uint32_t idesc_s = umma_idesc_f16(kRows, kBlk);
    constexpr uint32_t idesc_o = umma_idesc_f16(kRows, HD) | (1u << 16);  // B (V) MN-major
    const uint32_t q_addr = smem_addr(sQg), k_addr = smem_addr(sK), v_addr = smem_addr(sV), p_addr = smem_addr(sPg);
    const int row = gt;                        // query row of this thread (TMEM lane)
    const int qp = q0 + row;                   // its position in the prompt
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;

    for (int j = 0; j < nblk; ++j) {
        const int G = gb + j;  // global key-block index: barrier phases
        const int s = G & 1;
        // ---- S = Q K_j^T (K_{j+1} streams into the other stage once both groups' S_{G-1} retired)
        if (tid == 0 && j + 1 < nblk) {
            if (G >= 1) mbar_wait(&k_empty[s ^ 1], ((G - 1) >> 1) & 1);
            load_blk(j + 1, 0, sK + (s ^ 1) * C::kKV, &k_full[s ^ 1]);
        }
        if (gt == 0) {
            if (j == 0) mbar_wait(q_full, it & 1);
            mbar_wait(&k_full[s], (G >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < C::NH; ++c)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_bf16(tS, umma_desc_sw128(q_addr + c * C::kAtom + k * 32),
                              umma_desc_sw128(k_addr + s * C::kKV + c * C::kAtom + k * 32), idesc_s,
                              (c | k) != 0 ? 1u : 0u);
            umma_commit(s_done);
            umma_commit(&k_empty[s]);
        }
        mbar_wait(s_done, G & 1);
        tc_fence_after();
        // ---- softmax of this thread's row (two passes over TMEM: max, then exp/sum/P)
        const int kbase = j * kBlk;
        const int nvalid = min(kBlk, min(qp + 1, len) - kbase);  // keys [kbase, kbase + nvalid) are valid
        uint32_t r[32];
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            tmem_ld32(tS + lane_off + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (c * 32 + i < nvalid) mx = fmaxf(mx, __uint_as_float(r[i]));
        }
        const float m_new = fmaxf(m_run, mx * a.scale_log2);  // finite: key 0 of block 0 is valid
        const float alpha = fast_exp2(m_run - m_new);
        m_run = m_new;
        float rs = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            tmem_ld32(tS + lane_off + c * 32, r);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int k0 = c * 32 + 2 * i;
                const float p0 = k0 < nvalid ? fast_exp2(fmaf(__uint_as_float(r[2 * i]), a.scale_log2, -m_new)) : 0.f;
                const float p1 =
                    k0 + 1 < nvalid ? fast_exp2(fmaf(__uint_as_float(r[2 * i + 1]), a.scale_log2, -m_new)) : 0.f;
                rs += p0 + p1;
                pk[i] = pack_h2(p0, p1);
            }
            // keys [32c, 32c + 32): atom c / 2, 16 B chunks (c % 2) * 4 + q, XOR-swizzled by row
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int chunk = (c & 1) * 4 + q;
                const uint32_t dst = p_addr + (c >> 1) * C::kAtom + row * 128 + ((chunk ^ (row & 7)) << 4);
                asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(pk[4 * q]), "r"(pk[4 * q + 1]),
                             "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                             : "memory");
            }
        }
        l_run = l_run * alpha + rs;
        // ---- rescale O in place when a row's max moved (O of block j-1 is complete: o_done waited)
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
                tmem_ld32(tO + lane_off + c * 32, r);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                tmem_st32(tO + lane_off + c * 32, r);
            }
            tmem_st_wait();
        }
        fence_proxy_async_smem();  // P (generic-proxy stores) -> visible to the tensor core
        tc_fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");  // this group's 128 threads
        // ---- O += P V_j
        if (gt == 0) {
            mbar_wait(v_full, G & 1);
            tc_fence_after();
#pragma unroll
            for (int kc = 0; kc < kBlk / 16; ++kc)
                umma_bf16(tO, umma_desc_sw128(p_addr + (kc >> 2) * C::kAtom + (kc & 3) * 32),
                          umma_desc_sw128_mn(v_addr + kc * 2048, C::kAtom), idesc_o, (j | kc) != 0 ? 1u : 0u);
            umma_commit(o_done);
            umma_commit(v_empty);
        }
        mbar_wait(o_done, G & 1);  // this group's P and O are free again
        tc_fence_after();
        if (tid == 0 && j + 1 < nblk) {  // V_{j+1} once both groups' PV_j retired
            mbar_wait(v_empty, G & 1);
            load_blk(j + 1, 1, sV, v_full);
        }
    }

    // ---- epilogue: O / l -> bf16 (TMEM loads are warp-collective: every lane loads, rows past the prompt
    // do not store)
    {
        const float inv = 1.f / l_run;
        __nv_bfloat16* dst = out + (static_cast<long long>(start) + qp) * a.H * HD + static_cast<long long>(h) * HD;
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + lane_off + c * 32, r);
            tmem_ld_wait();
            if (qp < len) {
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    *reinterpret_cast<uint4*>(dst + c * 32 + v * 8) =
                        make_uint4(pack_bf2(__uint_as_float(r[8 * v]) * inv, __uint_as_float(r[8 * v + 1]) * inv),
                                   pack_bf2(__uint_as_float(r[8 * v + 2]) * inv, __uint_as_float(r[8 * v + 3]) * inv),
                                   pack_bf2(__uint_as_float(r[8 * v + 4]) * inv, __uint_as_float(r[8 * v + 5]) * inv),
                                   pack_bf2(__uint_as_float(r[8 * v + 6]) * inv, __uint_as_float(r[8 * v + 7]) * inv));
            }
        }
    }
    tc_fence_before();  // this item's O loads precede the group's next PV (ordered by its next bar.sync)
    gb += nblk;
    }  // items
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
}

template <int HD>
void tc_launch(const CUtensorMap& tq, const CUtensorMap& tkv, __nv_bfloat16* out, const PrefillTcArgs& a, int max_tiles,
               bool persistent, cudaStream_t st) {
    using C = TcCfg<HD>;
    static bool cfg = false;
    if (!cfg) {
        SW_CUDA(cudaFuncSetAttribute(attn_prefill_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        cfg = true;
    }
    // persistent: one CTA per SM of the stream's partition (smem and TMEM allow one), items round robin
    static const int persist_env = [] {  // SW_PREFILL_TC_PERSIST=0/1 forces (A/B); default: the caller's choice
        const char* v = std::getenv("SW_PREFILL_TC_PERSIST");
        return v && *v ? std::atoi(v) : -1;
    }();
    const bool persist = persist_env >= 0 ? persist_env != 0 : persistent;
    const int items = max_tiles * (a.H / 2);
    const int grid = std::max(1, persist ? std::min(items, stream_sm_count(st)) : items);
    launch_k(attn_prefill_tc_kernel<HD>, dim3(grid), dim3(256), C::kSmem, st, tq, tkv, out, a);
}

}  // namespace

void attn_prefill_tc(const CUtensorMap& tm_q, const CUtensorMap& tm_kv, __nv_bfloat16* out, const PrefillTcArgs& a,
                     int max_tiles, int hd, bool persistent, cudaStream_t st) {
    if (hd == 64) tc_launch<64>(tm_q, tm_kv, out, a, max_tiles, persistent, st);
    else if (hd == 128) tc_launch<128>(tm_q, tm_kv, out, a, max_tiles, persistent, st);
    else throw_cuda("attn_prefill_tc: head_dim must be 64 or 128", cudaErrorInvalidValue, __FILE__, __LINE__);
}

}  // namespace sw
