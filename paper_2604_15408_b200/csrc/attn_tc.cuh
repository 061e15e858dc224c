// attn_tc.cuh -- tcgen05 engine of the ragged attention (Alg. 1),
// included by kernels.cu (shares AttnArgs, image_rows, scan_cta_cu, TL).
//
// One CTA (4 warps) per (image, head), as in the mma.sync engine, but the two
// contractions run on the 5th-gen tensor cores with fp32 accumulators in TMEM:
//
//   S = Q K^T     tcgen05.mma kind::f16, M = 128 query rows, N = n16 keys, K = 64:
//                 A = Q tile, B = K rows, both SMEM (SWIZZLE_128B, K-major).
//   softmax       one thread per query row (TMEM lane): tcgen05.ld its S row,
//                 row max (no shuffles), P = 2^(S log2e/8 - m), row sum l;
//                 P is split hi + lo in the 16-bit type (R2) and written back
//                 with tcgen05.st IN PLACE of its S columns (2 values/column).
//   O = P V       tcgen05.mma with A = P from TMEM, B = V from SMEM (MN-major),
//                 N = 64, accumulated over all key chunks: P_hi V + P_lo V.
//   epilogue      tcgen05.ld O row, * 1/l, RNE to 16 bit, SMEM transpose,
//                 coalesced 128-byte row stores (scattered to padded rows).
//
// The whole sequence's S stays in TMEM (n <= 256 -> <= 256 columns) so the row
// max is final before any P is formed: the plain two-pass softmax the oracle
// defines, no online rescaling of O needed.  TMEM columns: 64 * ceil(n16/64)
// for S/P + 64 for O, rounded to a power of two (128 for n <= 64, the C3 case;
// 3 CTAs/SM then share 384 of the SM's 512 columns).  Queries beyond 128 rows
// (n > 128) run as a second M-tile reusing the same TMEM.
#pragma once

namespace ragged {

constexpr int kTcTile = 128;   // UMMA M: query rows per tile (one per thread)
constexpr int kTcChunk = 64;   // keys per softmax chunk = 64 fp32 TMEM columns

struct TcSmem {
  int kv_rows, off_q, off_k, off_v, off_small, bytes;
};
__host__ __device__ inline TcSmem tc_smem(int N) {
  TcSmem L;
  L.kv_rows = (N + 15) & ~15;
  L.off_q = 0;                                     // 128 x 128 B Q tile; O staging later
  L.off_k = kTcTile * kRowBytes;                   // kv_rows x 128 B, 1024-B aligned
  L.off_v = L.off_k + L.kv_rows * kRowBytes;
  L.off_small = L.off_v + L.kv_rows * kRowBytes;   // pos, drop, ballots, mbarriers, TMEM slot
  L.bytes = L.off_small + 2048 + 1024;             // + slack to align the base to 1024 B
  return L;
}

template <typename T, bool kFused>
__global__ void __launch_bounds__(kAttnThreads, 3) attn_tc_kernel(const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // SW128 atoms
  const TcSmem L = tc_smem(a.N);
  uint8_t* sQ = smem + L.off_q;
  uint8_t* sK = smem + L.off_k;
  uint8_t* sV = smem + L.off_v;
  uint8_t* small = smem + L.off_small;
  int16_t* sPos = reinterpret_cast<int16_t*>(small);
  int16_t* sDrop = sPos + kMaxN;
  uint32_t* sWords = reinterpret_cast<uint32_t*>(sDrop + kMaxN);
  uint64_t* bars = reinterpret_cast<uint64_t*>(small + 1088);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(small + 1104);
  const int tid = threadIdx.x, warp = tid >> 5;

  TL(0);
  int bid = blockIdx.x;
  if constexpr (kFused) {
    if (a.cu_out != nullptr) {
      if (bid == 0) {
        scan_cta_cu(a, sK);
        return;
      }
      bid -= 1;
    }
  }
  const int b = bid / a.H, h = bid - b * a.H;  // head fastest
  const long long HD = (long long)a.H * kHeadDim;
  int n;
  long long row_base;
  image_rows<kFused>(a, b, sPos, sDrop, sWords, n, row_base);

  const int ldb = (kFused ? (int)a.ld : (int)HD) * 2;
  const int HDb = (int)HD * 2;
  const char* img_q = static_cast<const char*>(a.q) + row_base * ldb + h * kRowBytes;
  const char* img_k = static_cast<const char*>(a.k) + row_base * ldb + h * kRowBytes;
  const char* img_v = static_cast<const char*>(a.v) + row_base * ldb + h * kRowBytes;
  char* img_o = static_cast<char*>(a.o) + row_base * HDb + h * kRowBytes + (tid & 7) * 16;

  auto zero_dropped = [&]() {  // dropped rows of this head -> +0.0
    if constexpr (kFused) {
      const int nd = a.N - n;
      const uint4 z = make_uint4(0u, 0u, 0u, 0u);
      for (int rr = tid >> 3; rr < nd; rr += kAttnThreads / 8) st_global_16(img_o + sDrop[rr] * HDb, z);
    }
  };
  if (n == 0) {  // nothing to attend (R11); returns before any TMEM allocation
    zero_dropped();
    return;
  }

  const int n16 = (n + 15) & ~15;
  const int nchunks = (n16 + kTcChunk - 1) / kTcChunk;  // 1..4
  const int o_col = nchunks * kTcChunk;                  // O columns after S/P
  const uint32_t ncols = o_col + 64 <= 128 ? 128u : (o_col + 64 <= 256 ? 256u : 512u);

  if (warp == 0) tc::alloc(smem_u32(tslot), ncols);
  if (tid == 32) {
    tc::mbar_init(smem_u32(&bars[0]), 1);
    tc::mbar_init(smem_u32(&bars[1]), 1);
    tc::fence_mbar_init();
  }

  // ---- stage K, V rows [0, n16) (zero past n: P = 0 there, V must be finite) ---
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
  auto load_q_tile = [&](int tile) {
    const int c = tid & 7, r0 = tid >> 3;
    const int rows = min(kTcTile, n - tile * kTcTile);
    const char* gsrc = img_q + c * 16;
    uint32_t sdst = smem_u32(sQ) + r0 * kRowBytes + ((c ^ (r0 & 7)) << 4);
    for (int rr = r0; rr < rows; rr += 16, sdst += 16 * kRowBytes)
      cp_async_16(sdst, gsrc + sPos[tile * kTcTile + rr] * ldb, 16);
  };
  load_q_tile(0);
  cp_async_commit();
  zero_dropped();  // overlaps the gathers in flight
  TL(2);
  cp_async_wait_all();
  tc::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  TL(3);

  const uint32_t tbase = *tslot;
  const uint32_t trow = tbase + ((uint32_t)(warp * 32) << 16);  // this warp's 32 lanes
  constexpr uint32_t kFmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
  const uint32_t idesc_s = tc::idesc_f16(kFmt, kTcTile, n16, 0);
  const uint32_t idesc_o = tc::idesc_f16(kFmt, kTcTile, kHeadDim, 1);
  const uint32_t bar_s = smem_u32(&bars[0]), bar_o = smem_u32(&bars[1]);
  constexpr float kScaleLog2 = 0.18033688011112042f;  // log2(e) / sqrt(64)
  uint32_t phase = 0;

  for (int tile = 0; tile * kTcTile < n; ++tile) {
    if (tile > 0) {
      load_q_tile(tile);
      cp_async_commit();
      cp_async_wait_all();
      tc::fence_proxy_async_smem();
      __syncthreads();
    }
    // ---- S = Q K^T: 4 UMMA of K = 16 (+32 B along the SW128 rows each) -------
    if (tid == 0) {
      tc::fence_after();
      const uint64_t qd = tc::sw128_desc(smem_u32(sQ)), kd = tc::sw128_desc(smem_u32(sK));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) tc::mma_ss(tbase, qd + 2 * kk, kd + 2 * kk, idesc_s, kk > 0);
      tc::commit(bar_s);
    }
    tc::mbar_wait(bar_s, phase);
    tc::fence_after();
    TL(5);

    // ---- softmax, one row per thread: pass A row max, pass B P (hi, lo) -> TMEM
    float m = -INFINITY;
    if (nchunks > 1) {
      for (int c0 = 0; c0 < n16; c0 += 32) {
        uint32_t r[32];
        tc::ld_x32(trow + c0, r);
        tc::wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < n) m = fmaxf(m, __uint_as_float(r[i]));
      }
    }
    float l = 0.f;
    for (int j = 0; j < nchunks; ++j) {
      const int c0 = j * kTcChunk;
      const bool two = c0 + 32 < n16;  // CTA-uniform
      uint32_t ra[32], rb[32];
      tc::ld_x32(trow + c0, ra);
      if (two) tc::ld_x32(trow + c0 + 32, rb);
      tc::wait_ld();
      if (nchunks == 1) {  // single chunk: the max comes from the same registers
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (c0 + i < n) m = fmaxf(m, __uint_as_float(ra[i]));
          if (two && c0 + 32 + i < n) m = fmaxf(m, __uint_as_float(rb[i]));
        }
      }
      const float ms = m * kScaleLog2;
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k0 = c0 + 2 * i;
        const float p0 = k0 < n ? ex2(__uint_as_float(ra[2 * i]) * kScaleLog2 - ms) : 0.f;
        const float p1 = k0 + 1 < n ? ex2(__uint_as_float(ra[2 * i + 1]) * kScaleLog2 - ms) : 0.f;
        l += p0 + p1;
        split2<T>(p0, p1, hi[i], lo[i]);
      }
      tc::st_x16(trow + c0, hi);        // P_hi keys c0..c0+31 -> cols c0 .. c0+15
      tc::st_x16(trow + c0 + 32, lo);   // P_lo               -> cols c0+32 .. c0+47
      if (two) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int k0 = c0 + 32 + 2 * i;
          const float p0 = k0 < n ? ex2(__uint_as_float(rb[2 * i]) * kScaleLog2 - ms) : 0.f;
          const float p1 = k0 + 1 < n ? ex2(__uint_as_float(rb[2 * i + 1]) * kScaleLog2 - ms) : 0.f;
          l += p0 + p1;
          split2<T>(p0, p1, hi[i], lo[i]);
        }
        tc::st_x16(trow + c0 + 16, hi);  // keys c0+32..c0+63 -> cols c0+16 .. c0+31
        tc::st_x16(trow + c0 + 48, lo);  //                   -> cols c0+48 .. c0+63
      }
    }
    tc::wait_st();
    tc::fence_before();
    __syncthreads();

    // ---- O = P_hi V + P_lo V over all key chunks (K = 16 keys per UMMA) -------
    if (tid == 0) {
      tc::fence_after();
      uint32_t acc = 0;
      for (int j = 0; j < nchunks; ++j) {
        const int nk = (min(kTcChunk, n - j * kTcChunk) + 15) >> 4;
        for (int kk = 0; kk < nk; ++kk) {
          const uint64_t vd = tc::sw128_desc(smem_u32(sV) + (j * kTcChunk + kk * 16) * kRowBytes);
          tc::mma_ts(tbase + o_col, tbase + j * kTcChunk + kk * 8, vd, idesc_o, acc);
          tc::mma_ts(tbase + o_col, tbase + j * kTcChunk + 32 + kk * 8, vd, idesc_o, 1u);
          acc = 1u;
        }
      }
      tc::commit(bar_o);
    }
    tc::mbar_wait(bar_o, phase);
    tc::fence_after();
    phase ^= 1u;

    // ---- epilogue: O / l -> 16 bit -> SMEM (sQ is free) -> 128-byte row stores
    {
      const float inv = 1.f / l;
      uint32_t oa[32], ob[32];
      tc::ld_x32(trow + o_col, oa);
      tc::ld_x32(trow + o_col + 32, ob);
      tc::wait_ld();
      uint8_t* srow = sQ + tid * kRowBytes;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t* s8 = c < 4 ? &oa[8 * c] : &ob[8 * (c - 4)];
        uint4 v;
        v.x = pack2<T>(__uint_as_float(s8[0]) * inv, __uint_as_float(s8[1]) * inv);
        v.y = pack2<T>(__uint_as_float(s8[2]) * inv, __uint_as_float(s8[3]) * inv);
        v.z = pack2<T>(__uint_as_float(s8[4]) * inv, __uint_as_float(s8[5]) * inv);
        v.w = pack2<T>(__uint_as_float(s8[6]) * inv, __uint_as_float(s8[7]) * inv);
        *reinterpret_cast<uint4*>(srow + ((c ^ (tid & 7)) << 4)) = v;
      }
    }
    tc::fence_before();
    __syncthreads();
    TL(6);
    {
      const int rows = min(kTcTile, n - tile * kTcTile);
      for (int rr = tid >> 3; rr < rows; rr += kAttnThreads / 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(sQ + rr * kRowBytes + (((tid & 7) ^ (rr & 7)) << 4));
        st_global_16(img_o + sPos[tile * kTcTile + rr] * HDb, v);
      }
    }
    __syncthreads();  // sQ and TMEM are reused by the next tile
  }
  if (warp == 0) {
    tc::fence_after();
    tc::dealloc(tbase, ncols);
  }
#ifdef RAGGED_TIMELINE
  __syncthreads();
  TL(4);
#endif
}

}  // namespace ragged
