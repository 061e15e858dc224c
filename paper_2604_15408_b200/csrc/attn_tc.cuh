// attn_tc.cuh -- tcgen05 engine of the ragged attention (Alg. 1),
// included by kernels.cu (shares AttnArgs, image_rows, scan_cta_cu, TL).
//
// Persistent CTAs, one per SM, each split into `nslots` (2-3) independent
// 128-thread SLOTS.  A slot processes one (image, head) problem at a time
// (problems are strided over CTAs then slots, head fastest as in P:293-294),
// in query tiles of 64 rows (16 per warp) and key chunks of 64:
//
//   S_j = Q K_j^T   tcgen05.mma kind::f16, M = 64, N <= 64 keys, K = 64; A = Q
//                   tile, B = K rows, both SMEM (SWIZZLE_128B, K-major); fp32
//                   accumulator in TMEM (tile row 16w + i -> lane 32w + i).
//   softmax         tcgen05.ld.16x256b: each thread holds rows g, g+8 of its
//                   warp's 16 and 2 of every 8 keys (the mma.sync fragment
//                   shape), 4 threads per row (quad shuffles for max / sum).
//                   Alg. 1's online update m, l, alpha with LAZY
//                   rescaling: the reference max only moves when a chunk max
//                   exceeds it by > 8 (log2), and then O is rescaled in TMEM.
//                   P = 2^(S log2e / 8 - m), split hi + lo in the 16-bit type
//                   (R2); the packed pair (keys 8j+2t, +1) is exactly what
//                   tcgen05.st.16x128b puts at P column 4j + t, so P lands IN
//                   PLACE of its S columns in the TS-UMMA A layout, no shuffles.
//   O += P_j V_j    tcgen05.mma with A = P from TMEM, B = V rows from SMEM
//                   (MN-major), N = 64: P_hi V + P_lo V.
//   epilogue        tcgen05.ld.16x256b the O rows, * 1/l, RNE to 16 bit, SMEM
//                   transpose, coalesced 128-byte row stores.
//
// TMEM: one 512-column allocation per CTA, issued before anything else (a
// resident tcgen05 CTA that has not yet allocated holds back the launch of the
// next CTA on its SM -- measured); each slot owns a fixed 128
// columns: S/P chunk [0, 64) + O [64, 128).  Warps whose 16 query rows are all
// padding skip the softmax and epilogue (and write the zero rows instead).
#pragma once

namespace ragged {

constexpr int kTcTile = 64;    // UMMA M: query rows per tile (16 per warp, 4 threads per row)
constexpr int kTcChunk = 64;   // keys per S/P chunk = 64 fp32 TMEM columns
constexpr int kTcSlotThreads = 128;

struct TcSmem {
  int kv_rows, off_q, off_k, off_v, off_small, slot_bytes;
};
// Per-slot layout (1024-B aligned SW128 tiles), then 1 KB of CTA-wide state.
__host__ __device__ inline TcSmem tc_smem(int N) {
  TcSmem L;
  L.kv_rows = (N + 15) & ~15;
  L.off_q = 0;                                     // 128 x 128 B: one Q tile or a tile pair; O staging later
  L.off_k = 2 * kTcTile * kRowBytes;               // kv_rows x 128 B
  L.off_v = L.off_k + L.kv_rows * kRowBytes;
  L.off_small = L.off_v + L.kv_rows * kRowBytes;   // pos, drop, ballots, scan scratch, mbarriers
  L.slot_bytes = L.off_small + 2048;
  return L;
}
__host__ __device__ inline int tc_smem_bytes(int N, int nslots) {
  return nslots * tc_smem(N).slot_bytes + 1024 /*CTA state*/ + 1024 /*alignment slack*/;
}
// Slots per CTA: as many as fit in the 227 KB per-CTA shared memory (max 3).
__host__ __device__ inline int tc_slots(int N) {
  for (int s = 3; s > 1; --s)
    if (tc_smem_bytes(N, s) <= 227 * 1024) return s;
  return 1;
}

template <typename T, bool kFused>
__global__ void __launch_bounds__(3 * kTcSlotThreads, 1) attn_tc_kernel(const AttnArgs a, int nwork) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nslots = blockDim.x / kTcSlotThreads;
  // warp-uniform slot / warp indices (UMMA operands then stay in uniform registers)
  const int wu = tc::warp_uniform_idx();
  const int slot = wu / (kTcSlotThreads / 32), tid = threadIdx.x % kTcSlotThreads;
  const int warp = wu % (kTcSlotThreads / 32);  // == CTA warp index % 4: this warp's TMEM lane quarter
  const TcSmem L = tc_smem(a.N);
  uint8_t* base = smem + slot * L.slot_bytes;
  uint8_t* sQ = base + L.off_q;
  uint8_t* sK = base + L.off_k;
  uint8_t* sV = base + L.off_v;
  uint8_t* small = base + L.off_small;
  int16_t* sPos = reinterpret_cast<int16_t*>(small);
  int16_t* sDrop = sPos + kMaxN;
  uint32_t* sWords = reinterpret_cast<uint32_t*>(sDrop + kMaxN);         // 32 B
  uint64_t* bars = reinterpret_cast<uint64_t*>(small + 1056);            // 6 x 8 B
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + nslots * L.slot_bytes);
  auto sync = [slot] { asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(kTcSlotThreads) : "memory"); };

  TL(0);
  pdl_launch_dependents();
  const uint32_t ncols_cta = nslots > 2 ? 512u : (nslots > 1 ? 256u : 128u);
  if (threadIdx.x < 32) tc::alloc(smem_u32(tslot), ncols_cta);  // first thing: see header
  if (tid == 32) {
    tc::mbar_init(smem_u32(&bars[0]), 1);  // single-tile path: S ready
    tc::mbar_init(smem_u32(&bars[1]), 1);  // single-tile path: P V done
    tc::mbar_init(smem_u32(&bars[2]), 1);  // pair path: tile A (S_{j+1} ready, P_j V_j done)
    tc::mbar_init(smem_u32(&bars[3]), 1);  // pair path: tile B
    bars[4] = 0ull;  // pair path: warps that stored P of tile A (atomic count, mod 4)
    bars[5] = 0ull;  // pair path: same for tile B
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_wait_prerequisites();  // TMEM/barrier setup above overlaps the previous grid's tail
  const uint32_t tbase = *tslot + (uint32_t)(slot * 128);        // this slot's 128 columns
  const uint32_t tS = tbase, tO = tbase + 64;
  // M = 64 accumulators: tile row 16w + i lives in TMEM lane 32w + i (i < 16)
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;          // this warp's lane quarter
  const int g = (tid & 31) >> 2, t4 = tid & 3;                     // fragment row / column pair
  const uint32_t bar_s = smem_u32(&bars[0]), bar_o = smem_u32(&bars[1]);
  uint32_t ph_s = 0, ph_o = 0;
  const uint32_t bar_x = smem_u32(&bars[2]);  // pair path: tile X uses bar_x + 8 X
  uint32_t ph_x[2] = {0u, 0u};                // pair path: per-tile barrier parities
  const uint32_t cnt_p = smem_u32(&bars[4]);  // pair path: P-stored counter of tile X at cnt_p + 8 X
  constexpr uint32_t kFmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
  const uint32_t idesc_o = tc::idesc_f16(kFmt, kTcTile, kHeadDim, 1);
  constexpr float kScaleLog2 = 0.18033688011112042f;  // log2(e) / sqrt(64)
  const long long HD = (long long)a.H * kHeadDim;
  const int HDb = (int)HD * 2;
  const int P = a.B * a.H;

  for (int w = blockIdx.x + gridDim.x * slot; w < nwork; w += gridDim.x * nslots) {
    if constexpr (kFused) {
      if (w == P) {  // the cu_seqlens work item (cu_mode 1 only)
        scan_cta_cu(a, sK, tid, sync);  // sK (>= 2 KB) is free during this item
        continue;
      }
    }
    const int b = w / a.H, h = w - b * a.H;
    int n;
    long long row_base;
    image_rows<kFused>(a, b, sPos, sDrop, sWords, n, row_base, tid, sync);

    const int ldb = (int)a.ld * 2;
    const char* img_q = static_cast<const char*>(a.q) + row_base * ldb + h * kRowBytes;
    const char* img_k = static_cast<const char*>(a.k) + row_base * ldb + h * kRowBytes;
    const char* img_v = static_cast<const char*>(a.v) + row_base * ldb + h * kRowBytes;
    char* img_o = static_cast<char*>(a.o) + row_base * HDb + h * kRowBytes + (tid & 7) * 16;
    // Dropped rows of this head -> +0.0, by threads [t0, t0 + nthr) of the slot.
    auto zero_dropped = [&](int t, int nthr) {
      if constexpr (kFused) zero_rows(img_o, sDrop, t >> 3, a.N - n, nthr >> 3, HDb);
    };
    // cu_mode 2: the head-0 problem of image b counts the keeps of images [0, b)
    // (while its gathers are in flight); reduced at the next slot barrier.
    const bool cu_here = kFused && a.cu_mode == 2 && h == 0;
    auto count_prefix = [&]() {
      int c = count_kept(a.keep, (long long)b * a.N, tid, kTcSlotThreads);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if ((tid & 31) == 0) sWords[warp] = (uint32_t)c;  // ballot words are dead now
    };
    auto write_cu = [&]() {  // after a slot barrier
      const int pre = (int)(sWords[0] + sWords[1] + sWords[2] + sWords[3]);
      a.cu_out[b] = pre;
      if (b == a.B - 1) a.cu_out[a.B] = pre + n;
    };
    if (n == 0) {  // nothing to attend (R11)
      if (cu_here) count_prefix();
      zero_dropped(tid, kTcSlotThreads);
      sync();      // sPos / sDrop are rewritten by the next problem
      if (cu_here && tid == 0) write_cu();
      sync();
      continue;
    }
    const int n16 = (n + 15) & ~15;
    const int nchunks = (n16 + kTcChunk - 1) / kTcChunk;

    // ---- stage K, V rows [0, n16) (zero past n: P = 0 there, V must be finite)
    {
      const int c = tid & 7, t = (tid >> 3) & 1, r0 = tid >> 4;
      const char* gsrc = (t ? img_v : img_k) + c * 16;
      uint32_t sdst = smem_u32(t ? sV : sK) + r0 * kRowBytes + ((c ^ r0) << 4);
      for (int r = r0; r < n16; r += 8, sdst += 8 * kRowBytes) {
        const bool valid = r < n;
        cp_async_16(sdst, gsrc + (valid ? sPos[r] * ldb : 0), valid ? 16 : 0);
      }
    }
    // Q tile rows [0, min(128, n - 128 tile)); rows past n stay unwritten: they
    // only feed their own (discarded) S / O rows.
    auto load_q_rows = [&](int first, int rows) {  // query rows [first, first+rows) -> sQ rows 0..
      const int c = tid & 7, r0 = tid >> 3;
      const char* gsrc = img_q + c * 16;
      uint32_t sdst = smem_u32(sQ) + r0 * kRowBytes + ((c ^ (r0 & 7)) << 4);
      for (int rr = r0; rr < rows; rr += 16, sdst += 16 * kRowBytes)
        cp_async_16(sdst, gsrc + sPos[first + rr] * ldb, 16);
    };
    auto load_q_tile = [&](int tile) { load_q_rows(tile * kTcTile, min(kTcTile, n - tile * kTcTile)); };
    load_q_rows(0, min(n, 2 * kTcTile));
    cp_async_commit();
    if (cu_here) count_prefix();
    TL(2);
    // warps [live, 4) own no query row of tile 0: they write the zero rows while
    // the others run the softmax; with no idle warp, every thread does it last.
    const int live = n >= kTcTile ? 4 : (n + 15) >> 4;

    // n > 64: query tiles processed in PAIRS inside the slot's 128 TMEM columns:
    // tile A (rows 128p .. +63) uses TMEM lanes 0-15 of each warp quarter, tile B
    // (rows 128p + 64 ..) lanes 16-31 (M = 64 UMMA at lane offset 16 -- verified,
    // scripts/micro/m64_lane16.cu).  The warps alternate the two tiles' softmax so
    // one tile's UMMAs run while the other's softmax executes; each tile's
    // S_{j+1} is queued right behind its P_j V_j, and one commit per tile and
    // chunk (tcgen05.commit tracks every prior UMMA of the thread) both signals
    // S_{j+1} and certifies P_j V_j, so lazy O-rescaling needs no extra wait.
    auto run_pairs = [&]() {
      const int npairs = (n + 2 * kTcTile - 1) / (2 * kTcTile);
      for (int pr = 0; pr < npairs; ++pr) {
        const int r0p = pr * 2 * kTcTile;
        const int rowsA = min(kTcTile, n - r0p), rowsB = max(0, min(kTcTile, n - r0p - kTcTile));
        const int ntl = rowsB > 0 ? 2 : 1;
        if (pr > 0) load_q_rows(r0p, rowsA + rowsB);
        cp_async_commit();
        cp_async_wait_all();
        tc::fence_proxy_async_smem();
        tc::fence_before();
        sync();
        tc::fence_after();
        if (pr == 0 && cu_here && tid == 0) write_cu();
        if (pr == 0) TL(3);
        if (pr == 0 && slot == 0) PT(0);
        float mm[2][2], ll[2][2];
#pragma unroll
        for (int X = 0; X < 2; ++X) mm[X][0] = mm[X][1] = -INFINITY, ll[X][0] = ll[X][1] = 0.f;
        // descriptors advance by bytes >> 4: a 64-row block of 128-byte rows = +512
        const uint64_t qd0 = tc::sw128_desc(smem_u32(sQ)), kd0 = tc::sw128_desc(smem_u32(sK));
        const uint64_t vd0 = tc::sw128_desc(smem_u32(sV));
        auto issue_s = [&](int X, int jj) {  // S of tile X, chunk jj
          const int kc = min(kTcChunk, n16 - jj * kTcChunk);
          tc::mma_ss_k64(tS + ((uint32_t)(16 * X) << 16), qd0 + 512ull * (uint64_t)X, kd0 + 512ull * (uint64_t)jj,
                         tc::idesc_f16(kFmt, kTcTile, kc, 0));
        };
        if (warp == 0) {
          if (tc::elect_one()) {
            for (int X = 0; X < ntl; ++X) {
              issue_s(X, 0);
              tc::commit(bar_x + 8u * (uint32_t)X);
            }
          }
          __syncwarp();
        }
        for (int j = 0; j < nchunks; ++j) {
          for (int X = 0; X < ntl; ++X) {
            tc::mbar_wait(bar_x + 8u * (uint32_t)X, ph_x[X]);
            ph_x[X] ^= 1u;
            tc::fence_after();
            if (pr == 0 && j == 0 && X == 0) TL(5);
            if (pr == 0 && slot == 0 && j < 4) PT(1 + 6 * j + 3 * X);
            const int rowsX = X ? rowsB : rowsA;
            if (warp * 16 < rowsX) {  // this warp owns real rows of tile X
              const uint32_t tSx = tS + lane_off + ((uint32_t)(16 * X) << 16);
              const uint32_t tOx = tO + lane_off + ((uint32_t)(16 * X) << 16);
              float& m0x = mm[X][0];
              float& m1x = mm[X][1];
              const int c0 = j * kTcChunk;
              const int nv = min(kTcChunk, n - c0);
              const int ngv = (nv + 7) >> 3;
              float x[8][4];
              {
                uint32_t r[32];
                tc::ld_16x256b_x8(tSx, r);
                tc::wait_ld();
#pragma unroll
                for (int jg = 0; jg < 8; ++jg)
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const int key = 8 * jg + 2 * t4 + (e & 1);
                    x[jg][e] = key < nv ? __uint_as_float(r[4 * jg + e]) * kScaleLog2 : -INFINITY;
                  }
              }
              float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
              for (int jg = 0; jg < 8; ++jg) {
                mx0 = fmaxf(mx0, fmaxf(x[jg][0], x[jg][1]));
                mx1 = fmaxf(mx1, fmaxf(x[jg][2], x[jg][3]));
              }
              mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
              mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
              mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
              mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
              float al0 = 1.f, al1 = 1.f;
              if (j == 0) {
                m0x = mx0;
                m1x = mx1;
              } else {
                if (mx0 - m0x > 8.f) { al0 = ex2(m0x - mx0); m0x = mx0; }
                if (mx1 - m1x > 8.f) { al1 = ex2(m1x - mx1); m1x = mx1; }
              }
              if (j > 0 && __any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {  // P_{j-1} V_{j-1} is done
                uint32_t o[32];
                tc::ld_16x256b_x8(tOx, o);
                tc::wait_ld();
#pragma unroll
                for (int jg = 0; jg < 8; ++jg) {
                  o[4 * jg + 0] = __float_as_uint(__uint_as_float(o[4 * jg + 0]) * al0);
                  o[4 * jg + 1] = __float_as_uint(__uint_as_float(o[4 * jg + 1]) * al0);
                  o[4 * jg + 2] = __float_as_uint(__uint_as_float(o[4 * jg + 2]) * al1);
                  o[4 * jg + 3] = __float_as_uint(__uint_as_float(o[4 * jg + 3]) * al1);
                }
                tc::st_16x256b_x8(tOx, o);
              }
              ll[X][0] *= al0;
              ll[X][1] *= al1;
              uint32_t hi[16], lo[16];
#pragma unroll
              for (int jg = 0; jg < 8; ++jg) {
                float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
                if (jg < ngv) {
                  p0 = ex2(x[jg][0] - m0x);
                  p1 = ex2(x[jg][1] - m0x);
                  p2 = ex2(x[jg][2] - m1x);
                  p3 = ex2(x[jg][3] - m1x);
                }
                ll[X][0] += p0 + p1;
                ll[X][1] += p2 + p3;
                split2<T>(p0, p1, hi[2 * jg], lo[2 * jg]);
                split2<T>(p2, p3, hi[2 * jg + 1], lo[2 * jg + 1]);
              }
              tc::st_16x128b_x8(tSx, hi);
              tc::st_16x128b_x8(tSx + 32, lo);
              tc::wait_st();
            }
            if (pr == 0 && slot == 0 && j < 4) PT(2 + 6 * j + 3 * X);
            // hand-off without waiting: each warp counts itself in once its P rows
            // are stored; the LAST warp to arrive issues P_j V_j (+ S_{j+1}) and
            // commits, so no warp ever blocks on the others' softmax and the
            // warps go straight on to the other tile.
            tc::fence_before();
            __syncwarp();
            uint32_t prev = 0;
            if ((tid & 31) == 0) {
              asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                           : "=r"(prev)
                           : "r"(cnt_p + 8u * (uint32_t)X)
                           : "memory");
            }
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if ((prev & 3u) == 3u) {  // P_j V_j for tile X, then S_{j+1} behind it
              tc::fence_after();
              const int nk = (min(kTcChunk, n - j * kTcChunk) + 15) >> 4;
              if (tc::elect_one()) {
                tc::mma_ts_pv(tO + ((uint32_t)(16 * X) << 16), tS + ((uint32_t)(16 * X) << 16),
                              vd0 + 512ull * (uint64_t)j, idesc_o, nk, j > 0 ? 1u : 0u);
                if (j + 1 < nchunks) issue_s(X, j + 1);
                tc::commit(bar_x + 8u * (uint32_t)X);
                if (pr == 0 && slot == 0 && j < 4) PT(3 + 6 * j + 3 * X);
              }
              __syncwarp();
            }
          }
        }
        if (pr == 0) TL(8);
        for (int X = 0; X < ntl; ++X) {  // the last commit certifies the last P V
          tc::mbar_wait(bar_x + 8u * (uint32_t)X, ph_x[X]);
          ph_x[X] ^= 1u;
        }
        tc::fence_after();
        if (pr == 0) TL(9);
        if (pr == 0 && slot == 0) PT(25);
        // epilogue: both tiles' O rows -> 16 bit -> SMEM (sQ is free) -> row stores
        for (int X = 0; X < ntl; ++X) {
          const int rowsX = X ? rowsB : rowsA;
          if (warp * 16 >= rowsX) continue;
          float l0 = ll[X][0], l1 = ll[X][1];
          l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
          l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
          l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
          l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
          const float inv0 = 1.f / l0, inv1 = 1.f / l1;
          uint32_t o[32];
          tc::ld_16x256b_x8(tO + lane_off + ((uint32_t)(16 * X) << 16), o);
          tc::wait_ld();
          const int r0 = X * kTcTile + warp * 16 + g, r1 = r0 + 8;
#pragma unroll
          for (int jg = 0; jg < 8; ++jg) {
            *reinterpret_cast<uint32_t*>(sQ + swz(r0, jg) + 4 * t4) =
                pack2<T>(__uint_as_float(o[4 * jg + 0]) * inv0, __uint_as_float(o[4 * jg + 1]) * inv0);
            *reinterpret_cast<uint32_t*>(sQ + swz(r1, jg) + 4 * t4) =
                pack2<T>(__uint_as_float(o[4 * jg + 2]) * inv1, __uint_as_float(o[4 * jg + 3]) * inv1);
          }
        }
        tc::fence_before();
        sync();
        for (int rr = tid >> 3; rr < rowsA + rowsB; rr += kTcSlotThreads / 8) {
          const uint4 v = *reinterpret_cast<const uint4*>(sQ + rr * kRowBytes + (((tid & 7) ^ (rr & 7)) << 4));
          st_global_16(img_o + sPos[r0p + rr] * HDb, v);
        }
        sync();  // sQ, TMEM reused by the next pair / problem
        if (pr == 0) TL(6);
        if (pr == 0 && slot == 0) PT(26);
        if (pr == 1 && slot == 0) PT(27);
      }
    };
    if (n > kTcTile) run_pairs();
    for (int tile = 0; n <= kTcTile && tile * kTcTile < n; ++tile) {
      if (tile > 0) load_q_tile(tile);
      cp_async_commit();
      cp_async_wait_all();
      tc::fence_proxy_async_smem();
      tc::fence_before();
      sync();
      TL(3);
      if (tile == 0 && cu_here && tid == 0) write_cu();
      // Warps [0, live_t) own real query rows of this tile and run the chunk loop;
      // the others skip straight to the store phase (on tile 0 they write the
      // zero rows meanwhile).  Inside the loop only the live warps synchronize.
      const int rows_t = n - tile * kTcTile;
      const int live_t = rows_t >= kTcTile ? 4 : (rows_t + 15) >> 4;
      const bool warp_live = warp < live_t;
      auto sync_live = [&] {
        asm volatile("bar.sync %0, %1;" ::"r"(4 + slot), "r"(live_t * 32) : "memory");
      };
      // Alg. 1 state for this thread's two rows g and g + 8 (log2 units); l is the
      // thread's partial row sum over its columns (quad-reduced at the end).
      float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
#ifndef RAGGED_TC_ZERO_LATE
      if (!warp_live && tile == 0) zero_dropped(tid - live * 32, (4 - live) * 32);
#endif

      for (int j = 0; warp_live && j < nchunks; ++j) {
        const int kc = min(kTcChunk, n16 - j * kTcChunk);     // keys in chunk (multiple of 16)
        // ---- S_j = Q K_j^T: 4 UMMA of K = 16 (+32 B along the SW128 rows each)
        if (warp == 0) {
          tc::fence_after();
          if (tc::elect_one()) {
            tc::mma_ss_k64(tS, tc::sw128_desc(smem_u32(sQ)), tc::sw128_desc(smem_u32(sK)) + 512ull * (uint64_t)j,
                           tc::idesc_f16(kFmt, kTcTile, kc, 0));
            tc::commit(bar_s);
          }
          __syncwarp();
        }
        tc::mbar_wait(bar_s, ph_s);
        ph_s ^= 1u;
        tc::fence_after();
        TL(5);

        {
          // S chunk in the accumulator fragment layout (16x256b): per 8-key group
          // jg, x[jg][0..1] = row g keys 8jg + 2t4 + {0,1}, x[jg][2..3] = row g + 8.
          const int c0 = j * kTcChunk;
          const int nv = min(kTcChunk, n - c0);  // valid keys in this chunk, >= 1
          const int ngv = (nv + 7) >> 3;         // 8-key groups holding valid keys
          float x[8][4];
          {
            uint32_t r[32];
            tc::ld_16x256b_x8(tS + lane_off, r);
            tc::wait_ld();
#pragma unroll
            for (int jg = 0; jg < 8; ++jg)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int key = 8 * jg + 2 * t4 + (e & 1);
                x[jg][e] = key < nv ? __uint_as_float(r[4 * jg + e]) * kScaleLog2 : -INFINITY;
              }
          }
          float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
          for (int jg = 0; jg < 8; ++jg) {
            mx0 = fmaxf(mx0, fmaxf(x[jg][0], x[jg][1]));
            mx1 = fmaxf(mx1, fmaxf(x[jg][2], x[jg][3]));
          }
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
          float al0 = 1.f, al1 = 1.f;
          if (j == 0) {
            m0 = mx0;
            m1 = mx1;
          } else {  // lazy: the reference max moves only if P would exceed 2^8
            if (mx0 - m0 > 8.f) { al0 = ex2(m0 - mx0); m0 = mx0; }
            if (mx1 - m1 > 8.f) { al1 = ex2(m1 - mx1); m1 = mx1; }
          }
          if (j > 0 && __any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {  // O *= alpha
            uint32_t o[32];
            tc::ld_16x256b_x8(tO + lane_off, o);
            tc::wait_ld();
#pragma unroll
            for (int jg = 0; jg < 8; ++jg) {
              o[4 * jg + 0] = __float_as_uint(__uint_as_float(o[4 * jg + 0]) * al0);
              o[4 * jg + 1] = __float_as_uint(__uint_as_float(o[4 * jg + 1]) * al0);
              o[4 * jg + 2] = __float_as_uint(__uint_as_float(o[4 * jg + 2]) * al1);
              o[4 * jg + 3] = __float_as_uint(__uint_as_float(o[4 * jg + 3]) * al1);
            }
            tc::st_16x256b_x8(tO + lane_off, o);
          }
          l0 *= al0;
          l1 *= al1;
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int jg = 0; jg < 8; ++jg) {  // P = e^{S - m}; groups past n skipped (exp2 unit)
            float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
            if (jg < ngv) {
              p0 = ex2(x[jg][0] - m0);
              p1 = ex2(x[jg][1] - m0);
              p2 = ex2(x[jg][2] - m1);
              p3 = ex2(x[jg][3] - m1);
            }
            l0 += p0 + p1;
            l1 += p2 + p3;
            // packed pair (keys 8jg + 2t4, +1) = P column 4jg + t4: the 16x128b store slot
            split2<T>(p0, p1, hi[2 * jg], lo[2 * jg]);
            split2<T>(p2, p3, hi[2 * jg + 1], lo[2 * jg + 1]);
          }
          tc::st_16x128b_x8(tS + lane_off, hi);       // P_hi: cols [0, 32) of the chunk
          tc::st_16x128b_x8(tS + lane_off + 32, lo);  // P_lo: cols [32, 64)
          tc::wait_st();
        }
        tc::fence_before();
        sync_live();
        TL(8);
        // ---- O += P_hi V_j + P_lo V_j (K = 16 keys per UMMA) --------------------
        if (warp == 0) {
          tc::fence_after();
          const int nk = (min(kTcChunk, n - j * kTcChunk) + 15) >> 4;
          if (tc::elect_one()) {
            tc::mma_ts_pv(tO, tS, tc::sw128_desc(smem_u32(sV)) + 512ull * (uint64_t)j, idesc_o, nk,
                          j > 0 ? 1u : 0u);
            tc::commit(bar_o);
          }
          __syncwarp();
        }
        tc::mbar_wait(bar_o, ph_o);  // before S_{j+1} overwrites P_j, and before the epilogue
        ph_o ^= 1u;
        tc::fence_after();
        TL(9);
      }

      if (!warp_live) {  // keep the mbarrier parities in step with the live warps
        ph_s ^= (uint32_t)(nchunks & 1);
        ph_o ^= (uint32_t)(nchunks & 1);
      }
      // ---- epilogue: O / l -> 16 bit -> SMEM (sQ is free) -> 128-byte row stores
      if (warp_live) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
        const float inv0 = 1.f / l0, inv1 = 1.f / l1;
        uint32_t o[32];
        tc::ld_16x256b_x8(tO + lane_off, o);
        tc::wait_ld();
        const int r0 = warp * 16 + g, r1 = r0 + 8;  // tile rows of this thread
#pragma unroll
        for (int jg = 0; jg < 8; ++jg) {  // dims 8jg + 2t4, +1 -> 4 bytes at chunk jg
          *reinterpret_cast<uint32_t*>(sQ + swz(r0, jg) + 4 * t4) =
              pack2<T>(__uint_as_float(o[4 * jg + 0]) * inv0, __uint_as_float(o[4 * jg + 1]) * inv0);
          *reinterpret_cast<uint32_t*>(sQ + swz(r1, jg) + 4 * t4) =
              pack2<T>(__uint_as_float(o[4 * jg + 2]) * inv1, __uint_as_float(o[4 * jg + 3]) * inv1);
        }
      }
      tc::fence_before();
      sync();
      TL(6);
      {
        const int rows = min(kTcTile, n - tile * kTcTile);
        for (int rr = tid >> 3; rr < rows; rr += kTcSlotThreads / 8) {
          const uint4 v = *reinterpret_cast<const uint4*>(sQ + rr * kRowBytes + (((tid & 7) ^ (rr & 7)) << 4));
          st_global_16(img_o + sPos[tile * kTcTile + rr] * HDb, v);
        }
      }
      sync();  // sQ, sPos, TMEM are reused by the next tile / problem
    }
#ifdef RAGGED_TC_ZERO_LATE
    if (true) {
#else
    if (live == 4) {
#endif
      zero_dropped(tid, kTcSlotThreads);
      sync();  // sDrop is rewritten by the next problem
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after();
    tc::dealloc(*tslot, ncols_cta);
  }
#ifdef RAGGED_TIMELINE
  TL(4);
#endif
}

}  // namespace ragged
