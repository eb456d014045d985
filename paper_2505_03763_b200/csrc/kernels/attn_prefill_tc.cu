// Prefill attention on the 5th-generation tensor cores (sm_100a tcgen05/TMEM).
//
// Causal flash attention for a varlen batch of prompts over the paged KV cache
// (GQA).  One work item = 128 query rows of one prompt for TWO query heads of
// the same kv head (they share every K/V block).  Warp-specialised CTA of 10
// warps:
//   warps 0-3 / 4-7   softmax of head 0 / head 1: thread t owns query row t
//                     (TMEM lane t); per 128-key block it tcgen05.ld's its S
//                     row ONCE (128 fp32 registers), takes the row max, writes
//                     P = exp2(S*scale - m) as fp16 back into TMEM over the
//                     first 64 columns of its own S accumulator, and arrives
//                     on p_full.  The running max is lazy: O and l are
//                     rescaled only when a block's max exceeds the max in use
//                     by more than 2^8 (P <= 256 then, exact in the final O/l);
//   warp 8            tcgen05.mma issuer (one thread):  S_g = Q_g K_j^T (SS,
//                     M=128 N=128 K=hd) and O_g += P_g V_j (TS: P from TMEM,
//                     V from smem as an MN-major B operand), in the order
//                     PV_0(j), S_0(j+1), PV_1(j), S_1(j+1): the tensor pipe
//                     runs one head's products while the other head's softmax
//                     runs.  S_g(j+1) overwrites P_g(j) only after PV_g(j) in
//                     the pipe's issue order;
//   warp 9            TMA producer: Q of both heads (3-D map over
//                     [tokens][H][hd]) and the K/V blocks, one 16-row box per
//                     page slice through the arena-wide map of the decode
//                     attention, into a ring of NS 128-key slots (K_0, Q, V_0,
//                     K_1, V_1, ...), so loads run several blocks ahead.
// TMEM (512 columns): S_0 [0,128), S_1 [128,256), O_0 [256,256+hd),
// O_1 [384,384+hd).  smem: Q (2 stages at hd 64) + the K/V ring, 193 KB (hd 64)
// / 225 KB (hd 128): one CTA per SM.  Items are dealt to a persistent grid (or
// one per CTA) last query tile first, snake order across rounds.
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

// 32 lanes x 16 32-bit columns, registers -> TMEM (P: 32 fp16 keys per thread per call).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]: the A operand (128 rows x 16 K, fp16 pairs per
// 32-bit column, K-major) read from tensor memory.
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int HD>
struct TcCfg {
    static constexpr int NH = HD / 64;           // 64-wide (128 B) column atoms of a head row
    static constexpr int kAtom = kRows * 128;    // one [128 rows][128 B] atom column
    static constexpr int kQ = NH * kAtom;        // one head's Q tile
    static constexpr int NQ = HD == 64 ? 2 : 1;  // Q stages (both heads per stage)
    static constexpr int kSlot = NH * kAtom;     // one K or V block of 128 keys
    static constexpr int NS = HD == 64 ? 8 : 5;  // K/V ring slots
    static constexpr int kOffRing = NQ * 2 * kQ;
    static constexpr int kOffBar = kOffRing + NS * kSlot;
    static constexpr int kSmem = 1024 + kOffBar + 256;
    static_assert(kSmem <= 227 * 1024, "smem budget");
    static constexpr uint32_t kTmemCols = 512;
    // warpgroups: softmax head 0 | softmax head 1 | MMA warp, TMA warp, two idle warps (setmaxnreg is
    // warpgroup-wide: the third group keeps 88 registers a thread and gives the rest to the softmax rows, 208 each)
    static constexpr int kThreads = 384;
};

// Work item k of CTA bx (both producer and consumers walk the same sequence).
struct Item {
    int tile, pair, start, len, q0, nblk, npages, pos0;
    const int32_t* ptab;
};
__device__ __forceinline__ bool next_item(const PrefillTcArgs& a, int k, Item& x) {
    const int pairs = a.H / 2;
    const int n_items = *a.n_tiles * pairs;
    const int G = static_cast<int>(gridDim.x), bx = static_cast<int>(blockIdx.x);
    const int idx = k * G + ((k & 1) ? G - 1 - bx : bx);
    if (idx >= n_items) return false;
    const int item = n_items - 1 - idx;  // last query tile first (most keys)
    x.tile = item / pairs;
    x.pair = item % pairs;
    const int sq = a.tile_seq[x.tile];
    x.q0 = a.tile_q0[x.tile];
    x.start = a.cu_seqlens[sq];
    x.len = a.cu_seqlens[sq + 1] - x.start;
    // a prompt chunk at positions [pos0, pos0 + len) attends to the cached prefix too; pos0 is a multiple
    // of 128, so the key blocks are aligned exactly as for a whole prompt and the last one is the diagonal
    x.pos0 = a.seq_pos0 ? a.seq_pos0[sq] : 0;
    const int kend = x.pos0 + min(x.q0 + kRows, x.len);  // keys this tile attends to: [0, kend)
    x.nblk = (kend + kBlk - 1) / kBlk;
    x.npages = (x.pos0 + x.len + kPg - 1) / kPg;
    x.ptab = a.page_table + static_cast<long long>(a.seq_slot[sq]) * a.max_pages;
    return true;
}

template <int HD>
__global__ void __launch_bounds__(384, 1) attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                              const __grid_constant__ CUtensorMap tm_kv,
                                                              __nv_bfloat16* __restrict__ out, PrefillTcArgs a) {
    using C = TcCfg<HD>;
    constexpr int NS = C::NS, NQ = C::NQ;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sRing = smem + C::kOffRing;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* q_full = bar;             // [NQ]
    uint64_t* q_empty = q_full + NQ;    // [NQ]  both heads' last S MMA of the item retired
    uint64_t* kv_full = q_empty + NQ;   // [NS]
    uint64_t* kv_empty = kv_full + NS;  // [NS]  both heads' MMAs reading the slot retired
    uint64_t* s_full = kv_empty + NS;   // [2]   S_g of the block in TMEM
    uint64_t* p_full = s_full + 2;      // [2]   P_g in TMEM (128 arrivals), O_g rescaled
    uint64_t* o_done = p_full + 2;      // [2]   the item's last PV_g retired
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NQ; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < NS; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&s_full[g], 1);
            mbar_init(&p_full[g], 128);
            mbar_init(&o_done[g], 1);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_kv);
    }
    if (warp == 8) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 9) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_last();  // K/V re-read by the prompt's later query tiles
            int n = 0, qi = 0;
            Item x{};
            // slot n of the ring <- K (v = 0) or V (v = 1) of key block j; page ids past the prompt read
            // page 0 (finite data, masked)
            auto load_slot = [&](int j, int v) {
                const int s = n % NS;
                if (n >= NS) mbar_wait(&kv_empty[s], ((n / NS) - 1) & 1);
                uint8_t* dst = sRing + s * C::kSlot;
                const int hk = (2 * x.pair) / (a.H / a.Hkv);
                int pid[kBlk / kPg];
#pragma unroll
                for (int i = 0; i < kBlk / kPg; ++i) {
                    const int pg = j * (kBlk / kPg) + i;
                    pid[i] = pg < x.npages ? x.ptab[pg] : 0;
                }
                mbar_expect_tx(&kv_full[s], C::kSlot);
#pragma unroll
                for (int i = 0; i < kBlk / kPg; ++i) {
                    const int kr = a.layer_row0 + pid[i] * a.page_rows + hk * kPg + (v ? a.v_rows : 0);
#pragma unroll
                    for (int c = 0; c < C::NH; ++c)
                        tma_load_2d(dst + c * C::kAtom + i * kPg * 128, &tm_kv, &kv_full[s], c * 64, kr, pol);
                }
                ++n;
            };
            for (int k = 0; next_item(a, k, x); ++k) {
                load_slot(0, 0);
                const int qs = qi % NQ;
                if (qi >= NQ) mbar_wait(&q_empty[qs], ((qi / NQ) - 1) & 1);
                mbar_expect_tx(&q_full[qs], 2 * C::kQ);
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int c = 0; c < C::NH; ++c)
                        tma_load_3d(sQ + (qs * 2 + g) * C::kQ + c * C::kAtom, &tm_q, &q_full[qs], c * 64,
                                    2 * x.pair + g, x.start + x.q0);
                ++qi;
                load_slot(0, 1);
                for (int j = 1; j < x.nblk; ++j) {
                    load_slot(j, 0);
                    load_slot(j, 1);
                }
            }
        }
        __syncwarp();
    } else if (warp == 8) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_s = umma_idesc_f16(kRows, kBlk);
            constexpr uint32_t idesc_o = umma_idesc_f16(kRows, HD) | (1u << 16);  // B (V) MN-major
            const uint32_t ring = smem_addr(sRing);
            int n = 0, qi = 0, gb = 0;
            Item x{};
            for (int k = 0; next_item(a, k, x); ++k) {
                const int qs = qi % NQ;
                mbar_wait(&q_full[qs], (qi / NQ) & 1);
                const uint32_t q_addr = smem_addr(sQ + qs * 2 * C::kQ);
                auto issue_s = [&](int g, int slot) {
                    const uint32_t kb = ring + slot * C::kSlot;
#pragma unroll
                    for (int c = 0; c < C::NH; ++c)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma_bf16(tmem + 128 * g, umma_desc_sw128(q_addr + g * C::kQ + c * C::kAtom + kk * 32),
                                      umma_desc_sw128(kb + c * C::kAtom + kk * 32), idesc_s, (c | kk) != 0 ? 1u : 0u);
                    umma_commit(&s_full[g]);
                };
                {
                    const int s = n % NS;
                    mbar_wait(&kv_full[s], (n / NS) & 1);
                    tc_fence_after();
                    issue_s(0, s);
                    issue_s(1, s);
                    umma_commit(&kv_empty[s]);
                    if (x.nblk == 1) umma_commit(&q_empty[qs]);
                }
                for (int j = 0; j < x.nblk; ++j) {
                    const int nv = n + 2 * j + 1, sv = nv % NS;
                    const int nk = nv + 1, sk = nk % NS;
                    const bool more = j + 1 < x.nblk;
                    mbar_wait(&kv_full[sv], (nv / NS) & 1);
                    const uint32_t vb = ring + sv * C::kSlot;
#pragma unroll
                    for (int g = 0; g < 2; ++g) {
                        mbar_wait(&p_full[g], (gb + j) & 1);
                        tc_fence_after();
#pragma unroll
                        for (int kc = 0; kc < kBlk / 16; ++kc)
                            umma_f16_ts(tmem + 256 + 128 * g, tmem + 128 * g + kc * 8,
                                        umma_desc_sw128_mn(vb + kc * 2048, C::kAtom), idesc_o, (j | kc) != 0 ? 1u : 0u);
                        if (more) {
                            if (g == 0) {
                                mbar_wait(&kv_full[sk], (nk / NS) & 1);
                                tc_fence_after();
                            }
                            issue_s(g, sk);
                        } else {
                            umma_commit(&o_done[g]);
                        }
                    }
                    umma_commit(&kv_empty[sv]);
                    if (more) {
                        umma_commit(&kv_empty[sk]);
                        if (j + 2 == x.nblk) umma_commit(&q_empty[qs]);
                    }
                }
                n += 2 * x.nblk;
                gb += x.nblk;
                ++qi;
            }
        }
        __syncwarp();
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
        // ------------------------------------------------------------ softmax (thread = query row)
        const int g = warp >> 2;
        const int row = tid & 127;
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + lane_off + 128 * g;  // S_g; P_g over its first 64 columns
        const uint32_t tO = tmem + lane_off + 256 + 128 * g;
        const float sl = a.scale_log2;
        int gb = 0, it = 0;
        Item x{};
        for (int k = 0; next_item(a, k, x); ++k) {
            const int h = 2 * x.pair + g;
            const int qr = x.q0 + row;    // this row in the prompt chunk
            const int qp = x.pos0 + qr;   // its position in the sequence
            float m_use = -INFINITY, l_run = 0.f;
            for (int j = 0; j < x.nblk; ++j) {
                mbar_wait(&s_full[g], (gb + j) & 1);
                tc_fence_after();
                uint32_t r[128];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
                tmem_ld_wait();
                // the diagonal / prompt-end block (the last): keys [kbase, kbase + nvalid) are valid
                const int nvalid = j + 1 == x.nblk ? min(kBlk, min(qp + 1, x.pos0 + x.len) - j * kBlk) : kBlk;
                float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
                for (int i = 0; i < 128; i += 2) {
                    if (i < nvalid) mx0 = fmaxf(mx0, __uint_as_float(r[i]));
                    if (i + 1 < nvalid) mx1 = fmaxf(mx1, __uint_as_float(r[i + 1]));
                }
                const float mb = fmaxf(mx0, mx1) * sl;  // finite: every row has a valid key in every block
                float alpha = 1.f;
                if (j == 0) {
                    m_use = mb;
                } else if (mb > m_use + 8.f) {  // lazy rescale: only when P would exceed 2^8
                    alpha = fast_exp2(m_use - mb);
                    m_use = mb;
                }
                if (__any_sync(0xffffffffu, alpha != 1.f)) {  // O_g is stable: PV_g(j-1) retired before S_g(j)
#pragma unroll
                    for (int c = 0; c < HD / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                        tmem_st32(tO + c * 32, o);
                    }
                }
                float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int k0 = 32 * c + 2 * i;
                        const float p0 = k0 < nvalid ? fast_exp2(fmaf(__uint_as_float(r[k0]), sl, -m_use)) : 0.f;
                        const float p1 = k0 + 1 < nvalid ? fast_exp2(fmaf(__uint_as_float(r[k0 + 1]), sl, -m_use)) : 0.f;
                        rs0 += p0;
                        rs1 += p1;
                        pk[i] = pack_h2(p0, p1);
                    }
                    tmem_st16(tS + c * 16, pk);
                }
                l_run = l_run * alpha + (rs0 + rs1);
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&p_full[g]);
            }
            // ---- epilogue: O / l -> bf16 (TMEM loads are warp-collective; rows past the prompt do not store)
            mbar_wait(&o_done[g], it & 1);
            tc_fence_after();
            const float inv = 1.f / l_run;
            __nv_bfloat16* dst = out + (static_cast<long long>(x.start) + qr) * a.H * HD + static_cast<long long>(h) * HD;
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_ld_wait();
                if (qr < x.len) {
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        *reinterpret_cast<uint4*>(dst + c * 32 + v * 8) =
                            make_uint4(pack_bf2(__uint_as_float(o[8 * v]) * inv, __uint_as_float(o[8 * v + 1]) * inv),
                                       pack_bf2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv),
                                       pack_bf2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv),
                                       pack_bf2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv));
                }
            }
            tc_fence_before();  // these O loads precede the next item's first PV (after this thread's p_full arrive)
            gb += x.nblk;
            ++it;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
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
    // persistent: one CTA per SM of the stream's partition (smem and TMEM allow one), items dealt round robin
    static const int persist_env = [] {  // SW_PREFILL_TC_PERSIST=0/1 forces (A/B); default: the caller's choice
        const char* v = std::getenv("SW_PREFILL_TC_PERSIST");
        return v && *v ? std::atoi(v) : -1;
    }();
    const bool persist = persist_env >= 0 ? persist_env != 0 : persistent;
    const int items = max_tiles * (a.H / 2);
    const int grid = std::max(1, persist ? std::min(items, stream_sm_count(st)) : items);
    launch_k(attn_prefill_tc_kernel<HD>, dim3(grid), dim3(C::kThreads), C::kSmem, st, tq, tkv, out, a);
}

}  // namespace

void attn_prefill_tc(const CUtensorMap& tm_q, const CUtensorMap& tm_kv, __nv_bfloat16* out, const PrefillTcArgs& a,
                     int max_tiles, int hd, bool persistent, cudaStream_t st) {
    if (hd == 64) tc_launch<64>(tm_q, tm_kv, out, a, max_tiles, persistent, st);
    else if (hd == 128) tc_launch<128>(tm_q, tm_kv, out, a, max_tiles, persistent, st);
    else throw_cuda("attn_prefill_tc: head_dim must be 64 or 128", cudaErrorInvalidValue, __FILE__, __LINE__);
}

}  // namespace sw
