// Persistent dataflow worker for a whole plan (see dataflow.hpp for the protocol).
//
// One CTA per SM, 12 warps:
//   8 consumer warps — DMMA k-tiles of GEMM items from the GEMM ring (common.cuh 3M k-tile,
//                      64 x 64 complex CTA tile, warp tile 32 x 16), epilogue, fused traces;
//   4 aux warps      — one per SM sub-partition; all lanes compute the TR_MM block pairs of
//                      the trace ring (8 rows of each 32 x 32 pair per warp, FP64 FMAs), and
//                      lane 0 of three of them carries a role:
//     issuer: streams operands of ready items through two TMA rings (GEMM, 64 KB stages: one
//       stage per 32-complex k-tile (A 64x32 + B 32x64 complex) or per partner tile of a fused
//       trace; trace, 32 KB stages: one 32x32 block pair A[t,I,J], B[t,J,I], 128-byte swizzled);
//       shared memory only, never blocks on global memory or on one ring;
//     GEMM / TR scheduler: claim items, decode them, poll their dependencies without
//       blocking, hand ready items to the issuer, and publish finished items (fence + done
//       counter).
// DMMA and DFMA share a sub-partition's FP64 pipe; trace FMAs in the aux warps take only
// their ~3 % share of it and never stall a warp that issues DMMAs.
// Reductions are deterministic: a chunked tile is summed chunk by chunk by the CTA that
// completes its last chunk (ticket); a TR_MM item's aux-warp partials are summed in warp order
// by the TR scheduler, and a slice's pieces in piece order by the CTA completing its last piece.
// Completion: the warps that worked on an item arrive on its done mbarrier after their stores
// (__syncwarp orders the lanes' stores first); the scheduler acquires it, fences at GPU scope
// (cumulative) and increments the op's done counter; a dependent CTA's scheduler acquires the
// counter (ld.acquire.gpu) and issues a proxy fence before TMA reads data other SMs wrote
// with ordinary stores.
#include "common.cuh"
#include "dataflow.hpp"
#include "kernels.hpp"

namespace cc {
namespace {
using namespace dev;

#ifndef DF_GSTAGES
#define DF_GSTAGES 2      // GEMM ring stages (64 KB at BK = 32)
#endif
#ifndef DF_TSTAGES
#define DF_TSTAGES 3      // trace ring stages (32 KB: one 32 x 32 complex block pair)
#endif
#ifndef DF_BK
#define DF_BK 32          // complex k per GEMM stage: 64 KB stages (12 TMA boxes per 64 KB instead
                          // of 10 per 32 KB at BK = 16; c2 3.73 -> 3.68 ms, c4 / c5 -1 to -2 %)
#endif
using GC = Cfg<64, 64, DF_BK, 32, 16, DF_GSTAGES>;   // (BK = 8: 16 KB stages with twice the barrier
                                                      // traffic measured 4.64-4.74 ms on c2; BK = 24 pads K = 128)
constexpr int CW = GC::NCW * 32;           // 256 consumer threads
#ifndef DF_NAUX
#define DF_NAUX 4         // trace warps (a multiple of 4: whole warpgroups, equal per sub-partition)
#endif
constexpr int NT = CW + 32 * DF_NAUX + 128;   // + trace warps + issuer, two schedulers, an idle warp
constexpr int TB = 32;                     // trace block edge (complex)
constexpr int INFO = 4;                    // item slots per queue (claimed-ready-running-unpublished)
constexpr int TSTAGE = 2 * TB * TB * 16;   // a trace block pair: A and B 32 x 32 complex (32 KB)
constexpr int TB_BYTES = TB * TB * 16;     // one operand block of a trace stage
// fused-trace partner stages (two halves of a 64 x 64 tile) need 32 or 64 KB GEMM stages
constexpr bool DF_FUSION = GC::STAGE_BYTES == TSTAGE || GC::STAGE_BYTES == 2 * TSTAGE;
constexpr int PHALF = GC::STAGE_BYTES / TSTAGE;       // partner-tile halves per GEMM stage (1 or 2)
constexpr int PSTAGES = PHALF >= 2 ? 1 : 2;           // GEMM stages per fused trace

__device__ __forceinline__ void tma_load_4d_g(void* dst, const void* map, uint64_t* bar, int c0, int c1, int c2,
                                              int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ double2 cmul_acc(double2 acc, double2 x, double2 y) {
  acc.x = fma(x.x, y.x, acc.x);
  acc.x = fma(-x.y, y.y, acc.x);
  acc.y = fma(x.x, y.y, acc.y);
  acc.y = fma(x.y, y.x, acc.y);
  return acc;
}

// One work item as the producer decoded it (shared memory, read by consumers and publisher).
struct ItemInfo {
  int64_t item;           // < 0: stop
  int64_t tile;           // GEMM
  const void* tA;
  const void* tB;
  int32_t op, kind, npos; // npos: stages the item consumes
  int32_t tm, tn, b, k0, kt_per_o, chunk;   // GEMM
  int32_t kt, fb, fc, ptmap0, rr;           // GEMM: k-tile stages, fused traces [fb, fb+fc) with
                                            // partner maps ptmap0.., tile index within its slice
  int32_t t, u0, nb, piece;                 // TRACE
  int32_t gj, gs;                           // TRACE: BB3 j extent and spin count (gj = 0: TR_MM)
  int32_t cw;                               // TRACE: chunk-wide maps (one box per operand block)
  unsigned long long t_disp, t_ready;       // profiling (producer)
  unsigned long long t_first, t_comp;       // profiling (consumers)
};

// Decode `item` of queue q.
__device__ __forceinline__ void decode_item(const DfQueue& q, int64_t item, ItemInfo& inf, const void* tmaps,
                                            const DfFused* fused) {
  inf.item = item;
  const int oi = q.item_op[item];
  const DfOp& op = q.ops[oi];
  const int64_t local = q.item_local[item];
  inf.op = oi;
  inf.kind = op.kind;
  inf.tA = static_cast<const uint8_t*>(tmaps) + size_t(2 * op.tmap) * 128;
  inf.tB = static_cast<const uint8_t*>(tmaps) + size_t(2 * op.tmap + 1) * 128;
  if (op.kind == 0) {
    const int64_t tile = local / op.n_chunks;
    const int chunk = int(local - tile * op.n_chunks);
    const int64_t tiles_mn = int64_t(op.tiles_m) * op.tiles_n;
    const int64_t b = tile / tiles_mn;
    const int64_t rr = tile - b * tiles_mn;
    inf.tile = tile;
    inf.chunk = chunk;
    inf.tn = int(rr / op.tiles_m);
    inf.tm = int(rr - int64_t(inf.tn) * op.tiles_m);
    inf.b = int(b);
    inf.k0 = int((int64_t(chunk) * op.KT) / op.n_chunks);
    inf.kt = int((int64_t(chunk + 1) * op.KT) / op.n_chunks) - inf.k0;
    inf.kt_per_o = op.kt_per_o;
    inf.rr = int(rr);
    inf.fb = op.fuse_begin;
    inf.fc = op.fuse_count;
    inf.ptmap0 = op.fuse_count > 0 ? fused[op.fuse_begin].tmap : 0;
    inf.npos = inf.kt + PSTAGES * op.fuse_count;   // + the partner stages of the fused traces
  } else {
    const int t = int(local / op.P), p = int(local - int64_t(t) * op.P);
    const int U = op.tr_G * op.nb * op.nb;
    inf.t = t;
    inf.piece = p;
    inf.nb = op.nb;
    inf.gj = op.tr_Gj;
    inf.gs = op.tr_S;
    inf.cw = op.tr_cw;
    inf.u0 = int((int64_t(p) * U) / op.P);
    inf.npos = int((int64_t(p + 1) * U) / op.P) - inf.u0;
  }
}

// Non-blocking dependency poll of an item working on time slice `slice`: advances *dep past
// satisfied dependencies.  A per-slice GEMM counter (target <= -2^20) is read at slot + slice.  A chunked copy (target -C) is needed only up to the chunk holding
// the slice: chunk k covers slices [k*Lt/C, (k+1)*Lt/C), so slice s is in chunk
// floor(((s+1)*C - 1) / Lt).
__device__ __forceinline__ bool deps_ready(const DfArgs& a, const DfOp& op, int slice, int* dep) {
  while (*dep < op.dep_count) {
    const int k = op.dep_begin + *dep;
    int target = a.dep_target[k];
    int slot = a.dep_slot[k];
    if (target <= -(1 << 20)) {
      slot += slice;
      target = -target - (1 << 20);
    } else if (target < 0) {
      target = int((int64_t(slice + 1) * (-target) - 1) / a.Lt) + 1;
    }
    if (ld_acquire(a.sync + slot) < target) return false;
    ++*dep;
  }
  return true;
}

#ifndef DF_TR_CW
#define DF_TR_CW 1        // TR_MM stages as one chunk-wide box per operand block (N % 8 == 0)
#endif
// Stage descriptor (producer -> consumers, one per ring stage)
constexpr uint32_t SK_STOP = 2;   // 0: data stage
constexpr uint32_t SD_FIRST = 1u << 5, SD_LAST = 1u << 6;
static_assert(INFO <= 8, "slot field is 3 bits");

__device__ __forceinline__ void gemm_stage_loads(const ItemInfo& inf, int k, uint8_t* sA, uint64_t* bar,
                                                 const void* tmaps) {
  using C = GC;
  if (k >= inf.kt) {
    // partner stage of fused trace f, half h: X[b, tn*64 + 32h + (0..31), tm*64 + (0..63)] as 8
    // boxes of 8 complex x 32 rows (row = j - 32h of the output tile, box c = columns i in
    // 8c..8c+7)
    // (a 64 KB stage holds both halves: h at byte offset h * 32 KB)
    const int f = (k - inf.kt) / PSTAGES;
    const void* map = static_cast<const uint8_t*>(tmaps) + size_t(2 * (inf.ptmap0 + f)) * 128;
    for (int h = PHALF >= 2 ? 0 : (k - inf.kt) & 1, hn = 0; hn < (PHALF >= 2 ? 2 : 1); ++h, ++hn)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        tma_load_4d_g(sA + hn * TSTAGE + c * 4096, map, bar, 2 * (inf.tm * C::BM + 8 * c), inf.tn * C::BN + 32 * h, 0,
                      inf.b);
    return;
  }
  uint8_t* sB = sA + C::A_BYTES;
  const int kk = inf.k0 + k;
  const int ko = kk / inf.kt_per_o;
  const int ki0 = (kk - ko * inf.kt_per_o) * C::BK;
#pragma unroll
  for (int kc = 0; kc < C::BK / 8; ++kc)
    tma_load_4d_g(sA + kc * C::BM * 128, inf.tA, bar, 2 * (ki0 + kc * 8), inf.tm * C::BM, ko, inf.b);
#pragma unroll
  for (int nc = 0; nc < C::BN / 8; ++nc)
    tma_load_4d_g(sB + nc * C::BK * 128, inf.tB, bar, 2 * (inf.tn * C::BN + nc * 8), ki0, ko, inf.b);
}

__device__ __forceinline__ void trace_stage_loads(const ItemInfo& inf, int k, uint8_t* sA, uint64_t* bar) {
  uint8_t* sB = sA + TB_BYTES;
  const int u = inf.u0 + k;
  const int nb2 = inf.nb * inf.nb;
  const int g = u / nb2, rem = u - g * nb2;
  const int I = rem / inf.nb, J = rem - I * inf.nb;
  if (inf.gj == 0 && inf.cw) {
    // one box per operand block: (16 doubles, 32 rows, 4 column chunks) lands as the same
    // [chunk][row][128 B] swizzled layout as four 32-row boxes
    tma_load_4d_g(sA, inf.tA, bar, 0, I * TB, J * (TB / 8), inf.t);
    tma_load_4d_g(sB, inf.tB, bar, 0, J * TB, I * (TB / 8), inf.t);
  } else if (inf.gj == 0) {
#pragma unroll
    for (int ch = 0; ch < TB / 8; ++ch) {  // A[t, I*32 + r, J*32 + 8ch + s] and B[t, J*32 + r, I*32 + 8ch + s]
      tma_load_4d_g(sA + ch * TB * 128, inf.tA, bar, 2 * (J * TB + 8 * ch), I * TB, 0, inf.t);
      tma_load_4d_g(sB + ch * TB * 128, inf.tB, bar, 2 * (I * TB + 8 * ch), J * TB, 0, inf.t);
    }
  } else {
    // BB3 sub-matrix g = (s, j): maps (k, j, row, t S + s) — the same 32 x 32 block pair layout
    const int j = g % inf.gj, ts = inf.t * inf.gs + g / inf.gj;
#pragma unroll
    for (int ch = 0; ch < TB / 8; ++ch) {
      tma_load_4d_g(sA + ch * TB * 128, inf.tA, bar, 2 * (J * TB + 8 * ch), j, I * TB, ts);
      tma_load_4d_g(sB + ch * TB * 128, inf.tB, bar, 2 * (I * TB + 8 * ch), j, J * TB, ts);
    }
  }
}

// Shared memory: the two dynamic rings (+ barriers + alignment slack) and the static control
// arrays (item slots, barriers, stage descriptors, trace partials) must fit 227 KB per CTA.
// The control arrays stay static: addressed through dynamic-region pointers they measured 2 %
// slower (c2: 4.75 vs 4.64 ms at 6 stages).
constexpr int GS = GC::STAGES;             // GEMM ring stages
constexpr int TS = DF_TSTAGES;             // trace ring stages
constexpr int STAGE = GC::STAGE_BYTES;     // GEMM stage (64 KB at BK = 32)
constexpr int DF_SMEM = GS * STAGE + TS * TSTAGE + 2 * (GS + TS) * 8 + 1024;
constexpr int DF_STATIC_SMEM =
    int(2 * INFO * sizeof(ItemInfo)) + 4 * INFO * 8 + (GS + TS) * 4 + INFO * DF_NAUX * 16 + 4;
static_assert(DF_SMEM + DF_STATIC_SMEM <= 232448, "dataflow worker exceeds 227 KB of shared memory");

// warp-uniform non-blocking mbarrier test (every lane tests; the warp agrees only when all see it)
__device__ __forceinline__ bool mbar_ready_warp(uint64_t* bar, uint32_t parity) {
  return __all_sync(0xffffffffu, mbar_test(bar, parity));
}

// Warps (16, four warpgroups): 8 consumer warps (DMMA k-tiles of the GEMM ring, warpgroups 0-1),
// 4 trace warps (warpgroup 2, one per SM sub-partition: the TR_MM block pairs of the trace
// ring, 8 rows of each 32 x 32 pair per warp) and warpgroup 3: issuer, GEMM scheduler, TR
// scheduler (lane 0 each) and an idle warp.  DMMA and DFMA share a sub-partition's FP64 pipe,
// so trace FMAs queue behind DMMAs: done by the consumer warps they stalled the warps issuing
// DMMAs (trace stages were 18.6 % of consumer time; interleaving their FMAs between DMMA
// k-quads, or running them in the role warps, measured slower still); in their own warps they
// take only their ~3 % share of the pipe.  Registers: launched at 128 per thread (512
// threads); setmaxnreg moves them to the consumers (184), from the trace warps (72) and the
// role warps (72) (no spills; 184 / 88 / 56 spilled in the role code).
// PROF: the instantiation with per-item / per-CTA timing (cc_execute flags bit 5); the plain
// one compiles every profiling statement out.
constexpr int NAUX = DF_NAUX;
static_assert(TB % NAUX == 0, "trace rows split evenly over the trace warps");
#ifndef DF_REG_MMA
#define DF_REG_MMA 184
#define DF_REG_TRACE 72
#define DF_REG_ROLE 72
#endif
constexpr int REG_MMA = DF_REG_MMA, REG_TRACE = DF_REG_TRACE, REG_ROLE = DF_REG_ROLE;
// setmaxnreg moves registers only within the CTA's launch allocation (NT x the launch count,
// a multiple of 8 per thread): the three budgets must fit in it, or setmaxnreg.inc never returns
constexpr int LAUNCH_REGS = (65536 / NT) / 8 * 8;
static_assert(8 * REG_MMA + NAUX * REG_TRACE + 4 * REG_ROLE <= (NT / 32) * LAUNCH_REGS,
              "register budgets exceed the CTA's launch allocation");
static_assert(NAUX % 4 == 0, "setmaxnreg works on whole warpgroups");
template <bool PROF>
__global__ void __launch_bounds__(NT, 1) df_worker(DfArgs a) {
  using C = GC;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned stage base, derived from the __shared__ array by pointer arithmetic so
  // the compiler keeps the shared address space (LDS, not generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* tsmem = smem + GS * STAGE;        // trace ring
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GS * STAGE + TS * TSTAGE);
  uint64_t* empty = full + GS;
  uint64_t* full_t = empty + GS;
  uint64_t* empty_t = full_t + TS;
  __shared__ ItemInfo s_info[2][INFO];
  __shared__ uint64_t info_full[2][INFO], done[2][INFO];
  __shared__ uint32_t s_desc[GS], s_desc_t[TS];
  __shared__ double2 red[INFO][NAUX];       // TR_MM item partials per trace warp, per slot
  __shared__ int s_flag;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < GS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    for (int s = 0; s < TS; ++s) {
      mbar_init(&full_t[s], 1);
      mbar_init(&empty_t[s], NAUX);
    }
    for (int s = 0; s < INFO; ++s) {
      mbar_init(&info_full[0][s], 1);     // scheduler -> issuer: item ready
      mbar_init(&info_full[1][s], 1);
      mbar_init(&done[0][s], C::NCW);     // consumers -> GEMM scheduler: item finished
      mbar_init(&done[1][s], NAUX);       // trace warps -> TR scheduler: trace item finished
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= C::NCW + NAUX) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_ROLE));
    const int role = warp - C::NCW - NAUX;   // 0 issuer, 1 GEMM scheduler, 2 TR scheduler, 3 idle
    if (lane != 0 || role == 3) return;
    // ---------------------------- issuer role (aux 0, lane 0) ------------------------------
    // Takes ready items of both kinds from the schedulers (shared memory only) and streams
    // their operands through the two TMA rings (GEMM: k-tiles and fused-trace partner tiles;
    // trace: block pairs); never blocks on global memory or on one ring while the other has
    // room.  Returns true once both rings carry their stop marker.
    uint32_t nx[2] = {0u, 0u}, pos[2] = {0u, 0u};
    bool have[2] = {false, false}, ex[2] = {false, false}, stop_put[2] = {false, false};
    int slot_of[2] = {0, 0}, k_of[2] = {0, 0}, np_of[2] = {0, 0};
    auto issuer_step = [&]() -> bool {
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (!have[x] && !ex[x]) {
          const int s = int(nx[x] % INFO);
          if (mbar_test(&info_full[x][s], (nx[x] / INFO) & 1u)) {
            ++nx[x];
            if (s_info[x][s].item < 0) {
              ex[x] = true;
            } else {
              have[x] = true;
              slot_of[x] = s;
              k_of[x] = 0;
              np_of[x] = s_info[x][s].npos;
            }
          }
        }
      }
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (!have[x] && !(ex[x] && !stop_put[x])) continue;
        const uint32_t nst = x ? uint32_t(TS) : uint32_t(GS);
        const int st = int(pos[x] % nst);
        if (!mbar_test(x ? &empty_t[st] : &empty[st], ((pos[x] / nst) & 1u) ^ 1u)) continue;
        uint32_t* desc = x ? &s_desc_t[st] : &s_desc[st];
        uint64_t* fb = x ? &full_t[st] : &full[st];
        ++pos[x];
        if (!have[x]) {                      // the queue is drained: the ring's stop marker
          *desc = SK_STOP;
          mbar_arrive(fb);
          stop_put[x] = true;
          continue;
        }
        const ItemInfo& inf = s_info[x][slot_of[x]];
        const int k = k_of[x];
        *desc = (uint32_t(slot_of[x]) << 2) | (k == 0 ? SD_FIRST : 0u) | (k == np_of[x] - 1 ? SD_LAST : 0u);
        mbar_expect_tx(fb, x ? TSTAGE : STAGE);
        if (x) trace_stage_loads(inf, k, tsmem + st * TSTAGE, fb);
        else gemm_stage_loads(inf, k, smem + st * STAGE, fb, a.tmaps);
        if (++k_of[x] == np_of[x]) have[x] = false;
      }
      return stop_put[0] && stop_put[1];
    };
    // ------------------ scheduler / publisher role (aux 1: GEMM, aux 2: TR, lane 0) --------
    // Claims items (at most `ahead` unpublished), decodes them, polls their dependencies
    // without blocking and hands ready items to the issuer in claim order; publishes finished
    // items in the same order (items of one kind finish in ring order): after the arrivals
    // on done[slot] (acquiring the stores) it makes the stores visible at GPU scope
    // (cumulative fence) and bumps the op's done counter, so neither the global-memory
    // latency of claiming and polling nor the fence's drain sits on the issuer's or the
    // consumers' path.  Returns true once the queue is drained and published.
    const int xq = role == 2 ? 1 : 0;
    const DfQueue& Q = xq == 0 ? a.q : a.qt;
    unsigned long long* prof = PROF ? (xq == 0 ? a.prof : a.prof_t) : nullptr;
    const uint32_t ahead = uint32_t(xq == 0 ? a.ahead_g : a.ahead_t);
    uint32_t n_alloc = 0, n_pub = 0;
    bool exhausted = Q.n_items == 0, pending = false, stopped = false;
    ItemInfo inf;
    int dep = 0;
    auto sched_step = [&]() -> bool {
      const int x = xq;
      while (n_pub < n_alloc && !(stopped && n_pub == n_alloc - 1)) {
        const int s = int(n_pub % INFO);
        if (!mbar_test(&done[x][s], (n_pub / INFO) & 1u)) break;
        const ItemInfo& cur = s_info[x][s];
        const DfOp& op = Q.ops[cur.op];
        if (x == 1) {
          // TR_MM piece: fixed-order sum of the trace warps' partials; a slice's pieces are
          // summed in piece order by the CTA that completes its last piece (ticket)
          double2 v = red[s][0];
#pragma unroll
          for (int w = 1; w < NAUX; ++w) {
            v.x += red[s][w].x;
            v.y += red[s][w].y;
          }
          double2* outp = static_cast<double2*>(op.out);
          if (op.P == 1) {
            outp[cur.t] = v;
          } else {
            double2* pp = static_cast<double2*>(op.tr_part) + int64_t(cur.t) * op.P;
            pp[cur.piece] = v;
            __threadfence();
            if (atomicAdd(&op.tr_cnt[cur.t], 1) == op.P - 1) {
              op.tr_cnt[cur.t] = 0;
              __threadfence();
              double2 sum = __ldcg(pp);
              for (int k = 1; k < op.P; ++k) {
                const double2 pk = __ldcg(pp + k);
                sum.x += pk.x;
                sum.y += pk.y;
              }
              outp[cur.t] = sum;
            }
          }
        }
        __threadfence();
        atomicAdd(a.sync + op.sync_id, 1);
        if (x == 0 && op.slice_sync >= 0) atomicAdd(a.sync + op.slice_sync + cur.b, 1);
        if (prof) {
          unsigned long long* pr = prof + 8 * cur.item;
          pr[0] = cur.t_disp;
          pr[1] = cur.t_ready;
          pr[2] = gtimer();
          pr[3] = smid();
          pr[4] = cur.t_first;
          pr[5] = cur.t_comp;
          pr[6] = uint64_t(x);
          pr[7] = cur.t_first;
        }
        ++n_pub;
      }
      if (stopped) return n_pub == n_alloc - 1;
      if (!pending && !exhausted && n_alloc - n_pub < ahead) {
        const unsigned long long t0 = prof ? gtimer() : 0ull;
        const int64_t it = int64_t(atomicAdd(Q.head, 1ull));
        if (it >= Q.n_items) {
          exhausted = true;
        } else {
          decode_item(Q, it, inf, a.tmaps, a.fused);
          inf.t_disp = t0;
          pending = true;
          dep = 0;
        }
      }
      if (pending && deps_ready(a, Q.ops[inf.op], x == 0 ? inf.b : inf.t, &dep)) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(inf.tA) : "memory");
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(inf.tB) : "memory");
        if (x == 0)
          for (int f = 0; f < inf.fc; ++f)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(
                             static_cast<const uint8_t*>(a.tmaps) + size_t(2 * (inf.ptmap0 + f)) * 128)
                         : "memory");
        inf.t_ready = prof ? gtimer() : 0ull;
        const int s = int(n_alloc % INFO);
        s_info[x][s] = inf;
        mbar_arrive(&info_full[x][s]);     // release: the item is visible to issuer and consumers
        ++n_alloc;
        pending = false;
      }
      if (!stopped && exhausted && !pending && n_alloc - n_pub < INFO) {
        const int s = int(n_alloc % INFO);
        s_info[x][s].item = -1;
        mbar_arrive(&info_full[x][s]);
        ++n_alloc;
        stopped = true;
      }
      return false;
    };
    if (role == 0) {
      while (!issuer_step()) {}
    } else {
      while (!sched_step()) __nanosleep(32);
    }
    return;
  }
  if (warp >= C::NCW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_TRACE));
    const int ax = warp - C::NCW;            // trace warp 0..3 (sub-partition ax)
    // ------------------------------------ trace rows -----------------------------------------
    // Rows ax, ax+4, ..., ax+28 of each 32 x 32 block pair, lane = column c: sum of
    // A[r][c] * B[c][r].  Element (row, col) of a block: chunk col/8, 128-byte row `row`,
    // 16-byte slot (col%8) ^ (row%8) (TMA 128-byte swizzle): A[r][c] row-contiguous, B[c][r]
    // one 128-byte row per lane — both conflict-free.  16 partial sums (4 row groups x the 4
    // real products of a complex MAC) keep the FMAs of one stage independent: they queue
    // behind the sub-partition's DMMAs, and nothing waits on them until the next stage.
#ifndef DF_TRG
#define DF_TRG 4
#endif
    constexpr int RG = DF_TRG;               // row groups of independent accumulators
    double accp[RG][4];
#pragma unroll
    for (int q = 0; q < RG; ++q) accp[q][0] = accp[q][1] = accp[q][2] = accp[q][3] = 0.0;
    uint32_t rt = 0;
    bool t_stop = false;
    long long n_tst = 0;
    // profile (trace warp 0, lane 0): cycles from the end of one stage until the next stage's
    // data is there (waiting for the issuer / TMA), and cycles computing stages
    long long tw_wait = 0, tw_work = 0, tw_mark = PROF ? clock64() : 0;
    // one trace stage if it is there; false when nothing was done
    auto trace_step = [&]() -> bool {
      if (t_stop) return false;
      const int st = int(rt % TS);
      if (!mbar_ready_warp(&full_t[st], (rt / TS) & 1u)) return false;
      const uint32_t d = s_desc_t[st];
      if ((d & 3u) == SK_STOP) {
        t_stop = true;
        return false;
      }
      long long tw0 = 0;
      if (PROF && lane == 0) {
        tw0 = clock64();
        tw_wait += tw0 - tw_mark;
      }
      if (d & SD_FIRST) {
#pragma unroll
        for (int q = 0; q < RG; ++q) accp[q][0] = accp[q][1] = accp[q][2] = accp[q][3] = 0.0;
        if (ax == 0 && lane == 0 && PROF) s_info[1][int((d >> 2) & 7u)].t_first = gtimer();
      }
      const uint8_t* sA = tsmem + st * TSTAGE;
      const uint8_t* sB = sA + TB_BYTES;
      const int c = lane;
#pragma unroll
      for (int qq = 0; qq < TB / NAUX; ++qq) {
        const int rr = ax + NAUX * qq;
        const double2 av = *reinterpret_cast<const double2*>(sA + (c >> 3) * (TB * 128) + rr * 128 +
                                                             (((c & 7) ^ (rr & 7)) << 4));
        const double2 bv = *reinterpret_cast<const double2*>(sB + (rr >> 3) * (TB * 128) + c * 128 +
                                                             (((rr & 7) ^ (c & 7)) << 4));
        double* p = accp[qq % RG];
        p[0] = fma(av.x, bv.x, p[0]);
        p[1] = fma(av.y, bv.y, p[1]);
        p[2] = fma(av.x, bv.y, p[2]);
        p[3] = fma(av.y, bv.x, p[3]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_t[st]);
      ++rt;
      if (PROF) ++n_tst;
      if (PROF && lane == 0) {
        tw_mark = clock64();
        tw_work += tw_mark - tw0;
      }
      if (d & SD_LAST) {
        const int slot = int((d >> 2) & 7u);
        if (ax == 0 && lane == 0 && PROF) s_info[1][slot].t_comp = gtimer();
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int q = 0; q < RG; ++q) {
          re += accp[q][0] - accp[q][1];
          im += accp[q][2] + accp[q][3];
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          re += __shfl_xor_sync(0xffffffffu, re, o);
          im += __shfl_xor_sync(0xffffffffu, im, o);
        }
        // the TR scheduler sums the trace warps' partials (fixed order) when it publishes
        if (lane == 0) red[slot][ax] = make_double2(re, im);
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[1][slot]);
      }
      return true;
    };
    for (;;) {
      if (!trace_step()) {
        if (t_stop) break;
        __nanosleep(20);
      }
    }
    if (PROF && lane == 0 && a.prof_sm) {
      a.prof_sm[16 * blockIdx.x + 8 + ax] = n_tst;
      if (ax == 0) {
        a.prof_sm[16 * blockIdx.x + 12] = tw_wait;
        a.prof_sm[16 * blockIdx.x + 13] = tw_work;
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_MMA));

  // ----------------------------------- consumers ---------------------------------------------
  // GEMM stages arrive in ring order; an item's stages are contiguous (k-tiles, then partner
  // stages of fused traces), and each item is processed by one block scope so its
  // accumulators (and the finished tile kept for fused traces) live only as long as the item.
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int g = lane >> 2, t = lane & 3;
  constexpr bool prof = PROF;
  // profile (thread 0): clock64 cycles waiting for stage data / in stage math, epilogue
  long long c_wait = 0, c_work = 0, n_st = 0, c_epi = 0, ta = 0, te = 0;
  uint32_t r = 0;
  auto next_stage = [&](int& st) -> uint32_t {
    st = int(r % GS);
    if (prof && tid == 0) ta = clock64();
    mbar_wait(&full[st], (r / GS) & 1u);
    if (prof && tid == 0) {
      c_wait += clock64() - ta;
      ++n_st;
    }
    ++r;
    return s_desc[st];
  };

  for (;;) {
    int st;
    uint32_t d = next_stage(st);
    if ((d & 3u) == SK_STOP) break;
    // ---------------- GEMM item: k-tiles, epilogue, then partner stages of fused traces ----------------
    const int slot = int((d >> 2) & 7u);
    const ItemInfo& cur = s_info[0][slot];
    if (tid == 0 && prof) s_info[0][slot].t_first = gtimer();
    {
      double acc[3][C::MI][C::NJ][2];   // 3M products (common.cuh dmma3m_ktile)
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NJ; ++j) acc[x][i][j][0] = acc[x][i][j][1] = 0.0;
      for (int k = 0;;) {
        const uint8_t* sA = smem + st * STAGE;
        if (prof && tid == 0) ta = clock64();
        dmma3m_ktile<C>(sA, sA + C::A_BYTES, wm, wn, g, t, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (prof && tid == 0) c_work += clock64() - ta;
        if (++k == cur.kt) break;
        d = next_stage(st);
      }
      if (prof && tid == 0) te = clock64();
      const DfOp& op = a.q.ops[cur.op];
      if (tid == 0 && prof) s_info[0][slot].t_comp = gtimer();
    const int64_t tile = cur.tile;
    const int chunk = cur.chunk;
    double2* out = static_cast<double2*>(op.C) + int64_t(cur.b) * op.sCb;
    // complex results C[row0 + 8i + g][col0 + 8j + 2t + e] = gauss3m_combine(acc, i, j, e)
    if (op.n_chunks == 1) {
      // lane (g, t) holds the adjacent complex columns 2t, 2t+1 of each 8-column block: one
      // 32-byte store (full sectors) when the row is 32-byte aligned and both columns exist
      const bool wide = (op.ldc & 1) == 0 && (op.sCb & 1) == 0 && (reinterpret_cast<uintptr_t>(op.C) & 31) == 0;
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        const int64_t row = int64_t(cur.tm) * C::BM + wm * C::WM + i * 8 + g;
        if (row >= op.M) continue;
#pragma unroll
        for (int j = 0; j < C::NJ; ++j) {
          const int64_t col = int64_t(cur.tn) * C::BN + wn * C::WN + j * 8 + 2 * t;
          const double2 v0 = gauss3m_combine<C>(acc, i, j, 0), v1 = gauss3m_combine<C>(acc, i, j, 1);
          double2* p = out + row * op.ldc + col;
          if (wide && col + 1 < op.Nn) {
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v0.x), "d"(v0.y), "d"(v1.x),
                         "d"(v1.y)
                         : "memory");
          } else {
            if (col < op.Nn) p[0] = v0;
            if (col + 1 < op.Nn) p[1] = v1;
          }
        }
      }
    } else {
      // publish this chunk's partial; the CTA completing the tile's last chunk sums them
      double2* base = static_cast<double2*>(op.part) + (tile * op.n_chunks) * int64_t(C::SLOT_DOUBLES / 2);
      double2* mine = base + int64_t(chunk) * (C::SLOT_DOUBLES / 2) + warp * (C::FRAG / 2 * 32);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            __stcg(mine + ((i * C::NJ + j) * 2 + e) * 32 + lane, gauss3m_combine<C>(acc, i, j, e));
      __threadfence();
      named_sync(1, CW);
      if (tid == 0) {
        const int old = atomicAdd(&op.tile_cnt[tile], 1);
        s_flag = (old == op.n_chunks - 1);
        if (s_flag) op.tile_cnt[tile] = 0;
      }
      named_sync(1, CW);
      if (s_flag) {
        __threadfence();
        const double2* w0 = base + warp * (C::FRAG / 2 * 32);
#pragma unroll
        for (int i = 0; i < C::MI; ++i) {
          const int64_t row = int64_t(cur.tm) * C::BM + wm * C::WM + i * 8 + g;
#pragma unroll
          for (int j = 0; j < C::NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int f = ((i * C::NJ + j) * 2 + e) * 32 + lane;
              double2 v = __ldcg(w0 + f);
              for (int c = 1; c < op.n_chunks; ++c) {
                const double2 u = __ldcg(w0 + int64_t(c) * (C::SLOT_DOUBLES / 2) + f);
                v.x += u.x;
                v.y += u.y;
              }
              const int64_t col = int64_t(cur.tn) * C::BN + wn * C::WN + j * 8 + 2 * t + e;
              if (row < op.M && col < op.Nn) out[row * op.ldc + col] = v;
            }
        }
      }
    }


      if (prof && tid == 0) c_epi += clock64() - te;
      if (cur.fc > 0) {
        // the tile's complex values stay in registers for the fused traces
        double2 v[C::MI][C::NJ][2];
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) v[i][j][e] = gauss3m_combine<C>(acc, i, j, e);
        for (int p = 0; p < PSTAGES * cur.fc; ++p) {
          d = next_stage(st);
          // partner half h (a 32 KB stage each, or both in one 64 KB stage) holds X rows j in [32h, 32h+32): the warps
          // whose output columns j fall there (wn = 2h, 2h+1: one warp per SM sub-partition)
          // add C[i][j] * X[j][i]; X[j][i] sits in box i/8 = 4wm + mi, row j - 32h, 16-byte
          // slot (i%8) ^ (j%8) = g ^ (2t+e) — conflict-free across each quarter warp
          const int f = p / PSTAGES, h = PHALF >= 2 ? (wn >> 1) : p & 1;
          if ((wn >> 1) == h) {
            const uint8_t* sP = smem + st * STAGE + (PHALF >= 2 ? h * TSTAGE : 0);
            double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < C::MI; ++i)
#pragma unroll
              for (int j = 0; j < C::NJ; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int jl = (wn & 1) * C::WN + 8 * j + 2 * t + e;   // row within the half
                  const double2 x = *reinterpret_cast<const double2*>(sP + (4 * wm + i) * 4096 + jl * 128 +
                                                                      ((g ^ (jl & 7)) << 4));
                  if (e == 0) s0 = cmul_acc(s0, v[i][j][e], x);
                  else s1 = cmul_acc(s1, v[i][j][e], x);
                }
            double2 sum = make_double2(s0.x + s1.x, s0.y + s1.y);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
              sum.x += __shfl_xor_sync(0xffffffffu, sum.x, o);
              sum.y += __shfl_xor_sync(0xffffffffu, sum.y, o);
            }
            if (lane == 0) {
              const DfFused& fz = a.fused[cur.fb + f];
              fz.part[(int64_t(cur.b) * fz.tiles + cur.rr) * C::NCW + warp] = sum;
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
        }
      }
    }
    // item finished: this warp's stores (ordered by __syncwarp) before the arrival
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[0][slot]);
  }
  if (prof && tid == 0 && a.prof_sm) {
    long long* ps = a.prof_sm + 16 * blockIdx.x;
    ps[0] = c_wait;
    ps[1] = 0;
    ps[2] = c_work;
    ps[3] = 0;
    ps[4] = n_st;
    ps[5] = 0;
    ps[6] = smid();
    ps[7] = c_epi;
  }
}

}  // namespace

namespace {
__global__ void fused_finish_kernel(const DfFused* __restrict__ fused, int64_t Lt);
}
cudaError_t df_preload() {
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, df_worker<false>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&attr, df_worker<true>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&attr, fused_finish_kernel);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(df_worker<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, DF_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(df_worker<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, DF_SMEM);
  return e;
}

void df_gemm_tile_dims(int* BM, int* BN, int* BK, int* slot_doubles) {
  *BM = GC::BM;
  *BN = GC::BN;
  *BK = GC::BK;
  *slot_doubles = GC::SLOT_DOUBLES;
}

int df_trace_block() { return TB; }

bool df_supports_fusion() { return DF_FUSION; }

cudaError_t df_launch(const DfArgs& a, int grid, cudaStream_t s) {
  if (a.prof) df_worker<true><<<grid, NT, DF_SMEM, s>>>(a);
  else df_worker<false><<<grid, NT, DF_SMEM, s>>>(a);
  return cudaGetLastError();
}

bool df_encode_maps(void* dst, const void* A, const void* B, int64_t M, int64_t Nn, int64_t Kin, int64_t Ko,
                    int64_t batch, int64_t lda, int64_t sAo, int64_t sAb, int64_t ldb, int64_t sBo, int64_t sBb) {
  ZgemmProblem p{};
  p.A = A;
  p.B = B;
  p.M = M;
  p.Nn = Nn;
  p.Kin = Kin;
  p.Ko = Ko;
  p.batch = batch;
  p.lda = lda;
  p.sAo = sAo;
  p.sAb = sAb;
  p.ldb = ldb;
  p.sBo = sBo;
  p.sBb = sBb;
  return encode_zgemm_maps(dst, static_cast<uint8_t*>(dst) + 128, p, GC::BM, GC::BK);
}

bool df_encode_partner_map(void* dst, const void* X, int64_t Lt, int64_t N) {
  // X as [Lt][N rows][N complex]: boxes of 32 rows x 8 complex (128-byte swizzle); the
  // second map of the pair is unused
  ZgemmProblem p{};
  p.A = X;
  p.B = X;
  p.M = N;
  p.Nn = N;
  p.Kin = N;
  p.Ko = 1;
  p.batch = Lt;
  p.lda = N;
  p.sAb = N * N;
  p.ldb = N;
  p.sBb = N * N;
  return encode_zgemm_maps(dst, static_cast<uint8_t*>(dst) + 128, p, TB, TB);
}

namespace {
__global__ void fused_finish_kernel(const DfFused* __restrict__ fused, int64_t Lt) {
  const DfFused& fz = fused[blockIdx.x];
  for (int64_t t = threadIdx.x; t < Lt; t += blockDim.x) {
    const double2* p = fz.part + t * fz.tiles * GC::NCW;
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < fz.tiles * GC::NCW; ++k) {   // tile-major, warp-minor: fixed order
      s.x += p[k].x;
      s.y += p[k].y;
    }
    fz.root[t] = s;
  }
}
}  // namespace

cudaError_t df_launch_fused_finish(const DfFused* fused, int32_t n_fused, int64_t Lt, cudaStream_t s) {
  if (n_fused <= 0) return cudaSuccess;
  fused_finish_kernel<<<unsigned(n_fused), 64, 0, s>>>(fused, Lt);
  return cudaGetLastError();
}

bool df_encode_bb3_maps(void* dst, const void* A, const void* B, int64_t Lt, int64_t N, int64_t S) {
  // X[t,s,r,j,c] (r = row of the sub-matrix, c = column) as dims (2N doubles of c, j, r, t S + s)
  const uint64_t dims[4] = {uint64_t(2 * N), uint64_t(N), uint64_t(N), uint64_t(Lt * S)};
  const uint64_t strides[3] = {uint64_t(N) * 16, uint64_t(N * N) * 16, uint64_t(N * N * N) * 16};
  const uint32_t box[4] = {16, 1, uint32_t(TB), 1};
  return encode_map_4d(dst, A, dims, strides, box) && encode_map_4d(static_cast<uint8_t*>(dst) + 128, B, dims, strides, box);
}

bool df_encode_trace_maps(void* dst, const void* A, const void* B, int64_t Lt, int64_t N, int32_t* chunk_wide) {
#if DF_TR_CW
  if (N % 8 == 0) {
    // A, B as 4-d views (16 doubles of a 128-byte column chunk, row, chunk, t): a box of
    // 16 x 32 x 4 is one 32 x 32 complex block, written to shared memory chunk-major (the
    // chunk stride, 128 B, is below the row stride: the view only reorders the box walk)
    const uint64_t dims[4] = {16, uint64_t(N), uint64_t(N / 8), uint64_t(Lt)};
    const uint64_t strides[3] = {uint64_t(N) * 16, 128, uint64_t(N * N) * 16};
    const uint32_t box[4] = {16, uint32_t(TB), uint32_t(TB / 8), 1};
    *chunk_wide = 1;
    return encode_map_4d(dst, A, dims, strides, box) && encode_map_4d(static_cast<uint8_t*>(dst) + 128, B, dims, strides, box);
  }
#endif
  *chunk_wide = 0;
  // A, B as [Lt][N rows][N complex]: boxes of 32 rows x 8 complex (128-byte swizzle)
  ZgemmProblem p{};
  p.A = A;
  p.B = B;
  p.M = N;
  p.Nn = N;
  p.Kin = N;
  p.Ko = 1;
  p.batch = Lt;
  p.lda = N;
  p.sAb = N * N;
  p.ldb = N;
  p.sBb = N * N;
  return encode_zgemm_maps(dst, static_cast<uint8_t*>(dst) + 128, p, TB, TB);
}

}  // namespace cc
