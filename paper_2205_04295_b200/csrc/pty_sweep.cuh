// pty_sweep.cuh -- the fused rPIE sweep: one cooperative persistent kernel per
// sweep (engine.py:173-243), all visits of all slots, no host round trips.
//
// Per visit step s (every slot advances to its position order[s]):
//   P1 rows  : gather o_j rows at the integer anchor (engine.py:192-195),
//              exit waves C*P_m*o_j for every mode (engine.py:113, C = (-1)^(r+c)),
//              forward row DFTs -> scratch;  max|o_j|^2 partials (engine.py:145)
//   P2 cols  : forward column DFTs (tile stays resident in shared memory),
//              max of total = sum_m |Psi_m|^2 partials (engine.py:114-117)
//   P3 cols  : modulus constraint scale = sqrt(I)/sqrt(total+eps) (engine.py:118),
//              error partials (engine.py:198-202), inverse column DFTs -> scratch
//   P4 rows  : inverse row DFTs -> corrected exit waves (engine.py:119),
//              rPIE object update (engine.py:123-137) written back with the
//              paste-add rounding (fields.py:101-107), rPIE probe update for every
//              mode with the pre-update crop (engine.py:140-150, 218-223), next
//              visit's max sum|P|^2 partials, posref staging (engine.py:226-230)
// separated by a software grid barrier.  The centered DFT of fields.py:71-84 is
// C * DFT(C * x) / W for even W, so no fftshift is materialised.
#pragma once
#include "pty_tasks.cuh"
#include "../../include/ptycho_b200.h"

namespace pty {

#ifdef PTY_NARROW256
constexpr int kSweepThreads = 512;     // narrow W = 256 lines: 32-lane groups, 128-thread teams
#else
constexpr int kSweepThreads = 256;
#endif
constexpr int kSweepMaxCtasPerSm = 2;
constexpr int kMaxSlots = 24;
constexpr int kStagedRows = 16;        // rows per staged P1/P4 task (one 128-byte scratch line per column)
constexpr int kMaxModes = 8;

struct SlotDev {
    void* obj;
    int H, Wc, r0, c0;
    void* probes;
    const void* patterns;
    const void* patterns_t;       // [N][W][W] each pattern transposed
    const double* positions;
    const int* order;
    void* stage;
    double* err_out;
    int* status;
};

struct SweepDev {
    int W, M, N, nslots;
    double alpha_o, alpha_p, beta, gamma, eps_rel;
    int update_probe, track_mod, sense;
    int resident;                 // P2 -> P3 column lines stay in shared memory (<= 1 column task per group)
    int p4_staged;                // P4: all modes' lines staged in shared memory, element-linear epilogue
    int p1_staged;                // P1: one task per row quad for all modes (needs p4_staged's shared memory)
    int slot_local;               // every phase's tasks of slot s live on CTAs [s*cps, (s+1)*cps): per-slot barriers
    int cps;                      // CTAs per slot (slot_local)
    unsigned int* slot_bar;       // [nslots][32] per-slot barrier counters (slot_local)
    int pair;                     // > 0: slots s and s + spp share the same SMs (virtual CTA index below)
    int pair_offset;              // > 0: slot s + spp starts after slot s finished this many phases
    unsigned int* sm_pair;        // [8 + 256]: SM-id bitmap, CTAs per SM (zeroed per launch)
    // workspace
    unsigned int* barrier;
    int* anchors;                 // [nslots][N][2]
    int4* steptab;                // [nslots][N]: (j, ar, ac, 0) of visit step t (order[t] and its anchor)
    void* scratch;                // [nslots][M][W][W] complex, transposed after the row pass
    void* totT;                   // [nslots][W][W] real
    void* omax_part;              // [2][nslots][W/4] real (by step parity)
    void* peak_part;              // [2][nslots][W/4] real
    void* tmax_part;              // [nslots][W] real
    double* err_part;             // [nslots][N][W][3] per-visit, per-column error terms
    void* ppg;                    // [nslots][W][W] real: sum_m |P_m|^2 of the current probes
    const void* twiddles;         // [W] complex, global
    unsigned long long* timeline; // debug: [steps][9][gridDim] globaltimer stamps or null
    int timeline_steps;
    // batched extension (oracle/batched.py contrib): slot s takes batch
    // positions k = s, s + nslots, ... (steptab (j, ar, ac, k), j < 0: idle
    // step); object and probes stay at the batch start; the P4->P1 barrier is
    // not needed (nothing a next step reads is written in P4)
    int batched;
    int visit0;                   // visit rank of batch position 0 (err_batch index)
    void* onum;                   // [b][W][W] complex: per-position object numerator
    void* pgroup;                 // [nslots][2M+1][W][W] real: per-slot probe numerators / denominator
    double* err_batch;            // [N_dataset][W][3] by visit rank
    SlotDev slot[kMaxSlots];
};

// shared-memory carve-up (bytes): twiddles | reduction scratch | phase region
template <typename T, int W>
__host__ __device__ constexpr size_t sweep_smem_fixed() {
    return (size_t)W * sizeof(cplx<T>) + 64 * sizeof(double);
}
// phase region: max over P1 (group exchange + team transpose tiles), P2/P3
// (group exchange) and P4 (team lines + per-team accumulators)
template <typename T, int W>
__host__ __device__ constexpr size_t sweep_smem_phase(int threads) {
    constexpr int B = Shape<W>::B, TEAM = 4 * B, XS = xch_size<W>(), LS4 = team_line_stride<W>();
    const int ngroups = threads / B, nteams = threads / TEAM;
    const size_t p1 = (size_t)ngroups * XS * sizeof(cplx<T>) + (size_t)nteams * W * 4 * sizeof(cplx<T>) +
                      (size_t)nteams * 4 * sizeof(T);
    const size_t p4 = (size_t)nteams * 4 * LS4 * sizeof(cplx<T>) + (size_t)nteams * 4 * W * sizeof(cplx<T>) +
                      (size_t)nteams * 4 * acc_stride<W>() * 2 * sizeof(T) + (size_t)nteams * 4 * sizeof(T);
    return p1 > p4 ? p1 : p4;
}

// Prefetch [base, base + bytes) into L2 (or L1 when to_l1), one request per
// 128-byte line, spread over the CTA's threads.
__device__ __forceinline__ void prefetch_span(const void* base, size_t bytes, bool to_l1) {
    const char* p = static_cast<const char*>(base);
    const size_t lines = (bytes + 127) / 128;
    for (size_t k = threadIdx.x; k < lines; k += blockDim.x) {
        if (to_l1) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + k * 128));
        else asm volatile("prefetch.global.L2 [%0];" ::"l"(p + k * 128));
    }
}

// Batched element copy: U independent loads in flight per thread before the
// stores (memory-level parallelism for L2-latency-bound tile moves).
template <int U, typename F>
__device__ __forceinline__ void batched(int n, F&& body) {
    for (int i0 = threadIdx.x; i0 < n; i0 += blockDim.x * U) body(i0);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// max over n partials, loaded by warp 0 in parallel and broadcast through
// shared memory.  Every thread of the CTA must call it.
template <typename T>
__device__ __forceinline__ T cta_max_of(const T* p, int n, T* cell) {
    if (threadIdx.x < 32) {
        T m = T(0);
        for (int i = threadIdx.x; i < n; i += 32) m = fmax(m, p[i]);
        m = warp_max(m);
        if (threadIdx.x == 0) *cell = m;
    }
    __syncthreads();
    const T v = *cell;
    __syncthreads();
    return v;
}

// One CTA's view of the sweep: shared-memory carve-up, per-thread constants
// and the four phases, one method per
// phase body; they are inlined (non-inlined member calls spill the CTA state
// to local memory, measured 2x slower).
//
// CL = false: one cooperative grid walks every slot in lock-step, phases
// separated by the software grid barrier.  CL = true: one thread-block cluster
// per slot (grid = nslots x clusterDim), phases separated by the hardware
// cluster barrier; slots run independently, so one slot's barrier wait is
// covered by another slot's CTAs on the same SM.
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_index() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
// all threads of all CTAs of the cluster; release/acquire at cluster scope
// orders the global-memory scratch traffic between phases
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <typename T, int W, bool CL, bool BAT = false>
__global__ void __launch_bounds__(kSweepThreads, kSweepMaxCtasPerSm) sweep_kernel(const __grid_constant__ SweepDev P) {
    using C = cplx<T>;
    constexpr int B = Shape<W>::B, TEAM = 4 * B, XS = xch_size<W>(), LS4 = team_line_stride<W>();
    constexpr int NTEAM = kSweepThreads / TEAM, NGRP = kSweepThreads / B;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // per-step snapshot of every slot: dead flag, position index, anchor
    __shared__ int s_dead[kMaxSlots], s_j[kMaxSlots], s_ar[kMaxSlots], s_ac[kMaxSlots], s_k[kMaxSlots];
    __shared__ unsigned long long s_mbar[NGRP];               // one bulk-copy barrier per line group
    unsigned mphase = 0u;                                      // its parity (identical on the group's lanes)
    C* tw = reinterpret_cast<C*>(smem_raw);
    T* red = reinterpret_cast<T*>(smem_raw + (size_t)W * sizeof(C));
    unsigned char* region = smem_raw + sweep_smem_fixed<T, W>();

    const int tid = threadIdx.x, NT = blockDim.x;
    const int M = P.M, N = P.N;
    // slot range and CTA coordinates of this kernel flavour
    const int s0 = CL ? (int)cluster_index() : 0;
    const int S = CL ? 1 : P.nslots;                       // slots walked by this CTA set
    const int cta = CL ? (int)cluster_rank() : (int)blockIdx.x;
    int vcta = cta;                                        // task-enumeration index (SM-paired in slot-local mode)
    const int ncta = CL ? (int)cluster_size() : (int)gridDim.x;
    const size_t WW = (size_t)W * W;
    // staged row tasks: blocks of RTS rows owned by a team of RTS groups
    constexpr int RTS = kStagedRows, TEAM_S = RTS * B, NTEAM_S = kSweepThreads / TEAM_S;
    constexpr int LSS = block_line_stride<W, RTS>();
    static_assert(kSweepThreads % TEAM_S == 0, "a staged team must divide the CTA");
    const int team_s = tid / TEAM_S, tl_s = tid % TEAM_S, gi_s = tl_s / B;
    const int rows_per_task = P.p4_staged ? RTS : 4;           // row tasks: blocks (staged) or quads
    const int nq = W / rows_per_task;
    const int team = tid / TEAM, tl = tid % TEAM, gi = tl / B, b = tid % B, grp = tid / B;
    const unsigned gmask = group_mask<W>();
    const UpdateParams U{P.alpha_o, P.alpha_p, P.beta, P.gamma, P.eps_rel, P.update_probe};
    C* scratch = reinterpret_cast<C*>(P.scratch);
    T* totT = reinterpret_cast<T*>(P.totT);
    T* omax_part = reinterpret_cast<T*>(P.omax_part);
    T* peak_part = reinterpret_cast<T*>(P.peak_part);
    T* tmax_part = reinterpret_cast<T*>(P.tmax_part);
    // phase-region views
    C* xch = reinterpret_cast<C*>(region) + grp * XS;                          // P1-P3
    C* res = reinterpret_cast<C*>(region) + (size_t)grp * P.M * XS;            // P2-P3 resident lines
    C* tt = reinterpret_cast<C*>(region) + (size_t)NGRP * XS + (size_t)team * W * 4;   // P1
    T* red4_p1 = reinterpret_cast<T*>(reinterpret_cast<C*>(region) + (size_t)NGRP * XS + (size_t)NTEAM * W * 4) + team * 4;
    C* lines = reinterpret_cast<C*>(region) + (size_t)team * 4 * LS4;                  // P4
    C* numer = reinterpret_cast<C*>(region) + (size_t)NTEAM * 4 * LS4 + (size_t)team * 4 * W;
    constexpr int RS = acc_stride<W>();
    T* acc_base = reinterpret_cast<T*>(reinterpret_cast<C*>(region) + (size_t)NTEAM * 4 * LS4 + (size_t)NTEAM * 4 * W);
    T* ppacc = acc_base + (size_t)team * 4 * RS;
    T* nppacc = acc_base + (size_t)NTEAM * 4 * RS + (size_t)team * 4 * RS;
    T* red4_p4 = acc_base + (size_t)2 * NTEAM * 4 * RS + team * 4;

    GridBarrier bar{P.barrier, 0u};
    // slot-local mode: after phase 0 a CTA only ever waits for the other CTAs
    // of its own slot (all of a slot's data -- scratch, canvas, probes,
    // partials -- is touched only by them), so slots drift independently and
    // a CTA waiting on its slot's barrier leaves the SM to the other slot's CTA
    bool local = false;
    unsigned int* my_bar = nullptr;
    unsigned int my_target = 0u;
    auto phase_sync = [&]() {
        if constexpr (CL) {
            cluster_sync();
        } else {
            if (local) {
                __syncthreads();
                my_target += (unsigned)P.cps;
                if (threadIdx.x == 0) {
                    unsigned int one = 1u, seen;
#ifdef PTY_BAR_RED
                    // arrival without a returned value: polling starts without
                    // waiting for the atomic's round trip
                    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(my_bar), "r"(one) : "memory");
#else
                    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(seen) : "l"(my_bar), "r"(one) : "memory");
#endif
                    while (true) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(my_bar) : "memory");
                        if ((int)(seen - my_target) >= 0) break;
#ifndef PTY_BAR_SPIN
                        __nanosleep(20);
#endif
                    }
                }
                __syncthreads();
            } else {
                bar.sync();
            }
        }
    };
    load_twiddles<T, W>(tw, reinterpret_cast<const C*>(P.twiddles));
    if (tid < NGRP) mbar_init(&s_mbar[tid], 1u);
    __syncthreads();

    // ---- phase 0: anchors (engine.py:69-70, 192-195) + bounds, initial probe peak
    for (int li = cta * NT + tid; li < (BAT ? 0 : S * N); li += ncta * NT) {
        const int idx = s0 * N + li;
        const int s = idx / N, j = idx % N;
        const SlotDev& sl = P.slot[s];
        const double x = sl.positions[2 * j], y = sl.positions[2 * j + 1];
        const int ar = (int)rint(y) - sl.r0;   // round half to even == Python round()
        const int ac = (int)rint(x) - sl.c0;
        P.anchors[2 * idx] = ar;
        P.anchors[2 * idx + 1] = ac;
        if (ar < 0 || ac < 0 || ar + W > sl.H || ac + W > sl.Wc) atomicOr(sl.status, PTY_ERR_BOUNDS);
        // step table: the visit at step t = j is order[t]; its anchor needs no second lookup
        const int t = j, jt = sl.order[t];
        const double xt = sl.positions[2 * jt], yt = sl.positions[2 * jt + 1];
        P.steptab[idx] = make_int4(jt, (int)rint(yt) - sl.r0, (int)rint(xt) - sl.c0, 0);
    }
    for (int item = cta; item < S * nq; item += ncta) {
        const int s = s0 + item / nq, rq = item % nq;
        const C* probes = reinterpret_cast<const C*>(P.slot[s].probes);
        T* ppg = reinterpret_cast<T*>(P.ppg) + (size_t)s * WW;
        T pk = T(0);
        for (int i = tid; i < rows_per_task * W; i += NT) {
            const size_t off = (size_t)(rows_per_task * rq) * W + i;
            T pp = T(0);
            for (int m = 0; m < M; ++m) pp += norm2(probes[m * WW + off]);
            ppg[off] = pp;
            pk = fmax(pk, pp);
        }
        pk = block_max(pk, red);
        if (tid == 0) peak_part[(size_t)s * nq + rq] = pk;
    }
    // SM pairing: register this CTA's SM (bitmap) and its rank among the CTAs on it
    __shared__ int s_vcta;
    unsigned my_sm = 0, my_rank = 0;
    if (!CL && P.pair > 0 && tid == 0) {
        asm volatile("mov.u32 %0, %%smid;" : "=r"(my_sm));
        my_sm &= 255u;
        atomicOr(&P.sm_pair[my_sm >> 5], 1u << (my_sm & 31));
        my_rank = atomicAdd(&P.sm_pair[8 + my_sm], 1u);
    }
    phase_sync();
    if constexpr (!CL) {
        if (P.slot_local) {
            // slots s and s + spp get the same SM set: virtual CTA = rank on the
            // SM * pair + dense index of the SM, so both CTAs of an SM serve the
            // same CTA position of two slots and every CTA of a slot sees the
            // same neighbour (uniform contention, balanced phases)
            if (P.pair > 0) {
                if (tid == 0) {
                    unsigned below = 0;
                    for (unsigned w = 0; w < (my_sm >> 5); ++w) below += __popc(P.sm_pair[w]);
                    below += __popc(P.sm_pair[my_sm >> 5] & ((1u << (my_sm & 31)) - 1u));
                    s_vcta = (my_rank < 2u && (int)below < P.pair) ? (int)my_rank * P.pair + (int)below : 0x3fffffff;
                }
                __syncthreads();
                vcta = s_vcta;
            }
            const int my_slot = vcta / P.cps;
            if (my_slot >= S) return;                          // idle CTA: no task in any phase
            local = true;
            my_bar = P.slot_bar + 32 * my_slot;
            // anti-phase start (PTY_SLOT_PAIR=2): the second slot on an SM set
            // begins once its partner slot has finished P1 and P2 of step 0, so
            // the two CTAs of an SM run different phases instead of the same
            const int spp = P.pair / P.cps;
            if (P.pair > 0 && P.pair_offset > 0 && my_slot >= spp && tid == 0) {
                const unsigned int* pb = P.slot_bar + 32 * (my_slot - spp);
                const unsigned int want = (unsigned)(P.pair_offset * P.cps);
                while (true) {
                    unsigned int seen;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(pb) : "memory");
                    if (seen >= want) break;
                    __nanosleep(100);
                }
            }
            __syncthreads();
        }
    }

    int4 v_next = make_int4(0, 0, 0, 0);
    if (tid < S) {
        v_next = P.steptab[(size_t)(s0 + tid) * N];
        s_dead[s0 + tid] = *(volatile const int*)P.slot[s0 + tid].status;   // phase-0 bounds errors
    }
    auto stamp = [&](int step, int k) {
        if (P.timeline && step < P.timeline_steps) {
            __syncthreads();
            if (tid == 0) P.timeline[((size_t)step * 9 + k) * gridDim.x + blockIdx.x] = gtimer();
        }
    };
    for (int step = 0; step < N; ++step) {
#ifdef PTY_PROBE
        if (blockIdx.x == 0 && tid == 0) pty_probe_step = step;
#endif
        stamp(step, 0);
        if (tid < S) {
            const int s = s0 + tid;
            // (j, ar, ac) of this step, loaded one step ahead (phase 0 wrote the table)
            const int4 v = v_next;
            if (step + 1 < N) v_next = P.steptab[(size_t)s * N + step + 1];
            // status only changes in P4 / phase 0, both behind a barrier.  In
            // slot-local mode a CTA tracks its own slot's P4 errors itself (all
            // of a slot's CTAs reduce the same maxima), so no reload per step
            if (!local) s_dead[s] = *(volatile const int*)P.slot[s].status;
            s_j[s] = v.x;
            s_ar[s] = v.y;
            s_ac[s] = v.z;
            s_k[s] = v.x < 0 ? -1 : v.w;                         // batched: -1 = no position this step
        }
        __syncthreads();
        // ---------------------------------------------------------- P1 rows
        if (P.p4_staged) {
            C* lines_m = reinterpret_cast<C*>(region) + (size_t)team_s * M * RTS * LSS;
            T* red_s = reinterpret_cast<T*>(reinterpret_cast<C*>(region) + (size_t)NTEAM_S * M * RTS * LSS) + team_s * RTS;
            for (int task = vcta * NTEAM_S + team_s; task < S * nq; task += ncta * NTEAM_S) {
                const int s = s0 + task / nq, rq = task % nq;
                if (s_dead[s] | (s_k[s] < 0)) continue;
                const SlotDev& sl = P.slot[s];
                const int j = s_j[s];
                const char* It = reinterpret_cast<const char*>(reinterpret_cast<const T*>(sl.patterns_t) + (size_t)j * WW +
                                                               (size_t)RTS * rq * W);
                for (int q = tl_s; q < (int)(RTS * W * sizeof(T) / 128); q += TEAM_S)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(It + q * 128));
                C* stg = P.sense == PTY_SENSE_XCORR_A ? reinterpret_cast<C*>(sl.stage) + (size_t)j * 2 * WW : nullptr;
                T om;
#define PTY_P1S(MM) om = task_rows_fwd_block<T, W, MM, RTS>(tw, lines_m, red_s, team_s, tl_s, gi_s, b, gmask, \
                    reinterpret_cast<const C*>(sl.obj), sl.Wc, s_ar[s], s_ac[s], reinterpret_cast<const C*>(sl.probes), rq, \
                    scratch + (size_t)s * M * WW, stg)
                switch (M) {
                    case 1: PTY_P1S(1); break;
                    case 2: PTY_P1S(2); break;
                    case 3: PTY_P1S(3); break;
                    default: PTY_P1S(4); break;
                }
#undef PTY_P1S
                if (tl_s == 0) omax_part[((size_t)(step & 1) * P.nslots + s) * nq + rq] = om;
            }
        } else
        for (int task = vcta * NTEAM + team; task < S * M * nq; task += ncta * NTEAM) {
            const int s = s0 + task / (M * nq), m = (task / nq) % M, rq = task % nq;
            if (s_dead[s] | (s_k[s] < 0)) continue;
            const SlotDev& sl = P.slot[s];
            const int j = s_j[s];
            // this visit's pattern column lines P3 will read: HBM -> L2
            if (m == 0) {
                const char* It = reinterpret_cast<const char*>(reinterpret_cast<const T*>(sl.patterns_t) + (size_t)j * WW +
                                                               (size_t)4 * rq * W);
                for (int q = tl; q < (int)(4 * W * sizeof(T) / 128); q += TEAM)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(It + q * 128));
            }
            C* stg = (P.sense == PTY_SENSE_XCORR_A && m == 0) ? reinterpret_cast<C*>(sl.stage) + (size_t)j * 2 * WW : nullptr;
            const T om = task_row_fwd<T, W>(tw, xch, tt, red4_p1, team, tl, gi, b, gmask,
                                            reinterpret_cast<const C*>(sl.obj), sl.Wc, s_ar[s], s_ac[s],
                                            reinterpret_cast<const C*>(sl.probes), m, rq, scratch + (size_t)s * M * WW, stg);
            if (m == 0 && tl == 0) omax_part[((size_t)(step & 1) * P.nslots + s) * nq + rq] = om;
        }
        stamp(step, 1);
        phase_sync();
        stamp(step, 2);
        // ------------------------------------------------- P2 cols (forward)
        for (int task = vcta * NGRP + grp; task < S * W; task += ncta * NGRP) {
            const int s = s0 + task / W, kc = task % W;
            if (s_dead[s] | (s_k[s] < 0)) continue;
            const T tm = P.resident
                ? task_col_fwd<T, W, true>(tw, xch, b, gmask, scratch + (size_t)s * M * WW, M, kc, totT + (size_t)s * WW, res,
                                           &s_mbar[grp], &mphase)
                : task_col_fwd<T, W, false>(tw, xch, b, gmask, scratch + (size_t)s * M * WW, M, kc, totT + (size_t)s * WW);
            if (b == 0) tmax_part[(size_t)s * W + kc] = tm;
        }
        stamp(step, 3);
        phase_sync();
        stamp(step, 4);
        // ---------------------------------------- P3 modulus + cols (inverse)
        for (int task = vcta * NGRP + grp; task < S * W; task += ncta * NGRP) {
            const int s = s0 + task / W, kc = task % W;
            if (s_dead[s] | (s_k[s] < 0)) continue;
            const SlotDev& sl = P.slot[s];
            const int j = s_j[s];
            C* stg = P.sense == PTY_SENSE_XCORR_B ? reinterpret_cast<C*>(sl.stage) + (size_t)j * 2 * WW : nullptr;
            const T* It = reinterpret_cast<const T*>(sl.patterns_t) + (size_t)j * WW;
            double* ep = BAT ? P.err_batch + ((size_t)(P.visit0 + s_k[s]) * W + kc) * 3
                                   : P.err_part + (((size_t)s * N + step) * W + kc) * 3;
            if (P.resident)
                task_col_mod<T, W, true>(tw, xch, b, gmask, scratch + (size_t)s * M * WW, M, kc, totT + (size_t)s * WW,
                                         tmax_part + (size_t)s * W, It, T(P.eps_rel), P.track_mod, stg, ep, res);
            else
                task_col_mod<T, W, false>(tw, xch, b, gmask, scratch + (size_t)s * M * WW, M, kc, totT + (size_t)s * WW,
                                          tmax_part + (size_t)s * W, It, T(P.eps_rel), P.track_mod, stg, ep);
        }
        stamp(step, 5);
        phase_sync();
        stamp(step, 6);
        // --------------------------------------- P4 rows (inverse) + update
        if (P.p4_staged) {
            C* lines_m = reinterpret_cast<C*>(region) + (size_t)team_s * M * RTS * LSS;
            T* red_s = reinterpret_cast<T*>(reinterpret_cast<C*>(region) + (size_t)NTEAM_S * M * RTS * LSS) + team_s * RTS;
            for (int task = vcta * NTEAM_S + team_s; task < S * nq; task += ncta * NTEAM_S) {
                const int s = s0 + task / nq, rq = task % nq;
                if (s_dead[s] | (s_k[s] < 0)) continue;
                const SlotDev& sl = P.slot[s];
                const int j = s_j[s];
                // the maxima partials are reduced inside the task, while the
                // block's scratch rows are already in flight (engine.py:132-134,
                // 145-147 checked there: a failing slot returns its error bit)
                const T* pkp = peak_part + ((size_t)(BAT ? 0 : step & 1) * P.nslots + s) * nq;
                const T* omp = omax_part + ((size_t)(step & 1) * P.nslots + s) * nq;
                int bad = 0;
                if constexpr (BAT) {
#define PTY_P4A(MM) task_rows_acc_block<T, W, MM, RTS>(tw, lines_m, team_s, tl_s, gi_s, b, gmask, \
                    scratch + (size_t)s * M * WW, rq, reinterpret_cast<const C*>(sl.obj), sl.Wc, s_ar[s], s_ac[s], \
                    reinterpret_cast<const C*>(sl.probes), pkp, omp, nq, U, reinterpret_cast<C*>(P.onum) + (size_t)s_k[s] * WW, \
                    reinterpret_cast<T*>(P.pgroup) + (size_t)s * (2 * M + 1) * WW, bad)
                    switch (M) {
                        case 1: PTY_P4A(1); break;
                        case 2: PTY_P4A(2); break;
                        case 3: PTY_P4A(3); break;
                        default: PTY_P4A(4); break;
                    }
#undef PTY_P4A
                    if (bad) {
                        if (tl_s == 0) atomicOr(sl.status, bad);
                        if (local && tid == 0) s_dead[s] = 1;
                    }
                } else {
                C* stg = P.sense == PTY_SENSE_XCORR_A ? reinterpret_cast<C*>(sl.stage) + (size_t)j * 2 * WW : nullptr;
                T npk;
#define PTY_P4S(MM) npk = task_rows_inv_block<T, W, MM, RTS>(tw, lines_m, red_s, team_s, tl_s, gi_s, b, gmask, \
                    scratch + (size_t)s * M * WW, rq, reinterpret_cast<C*>(sl.obj), reinterpret_cast<T*>(P.ppg) + (size_t)s * WW, \
                    sl.Wc, s_ar[s], s_ac[s], reinterpret_cast<C*>(sl.probes), pkp, omp, nq, U, stg, bad)
                switch (M) {
                    case 1: PTY_P4S(1); break;
                    case 2: PTY_P4S(2); break;
                    case 3: PTY_P4S(3); break;
                    default: PTY_P4S(4); break;   // host enables staging only for M <= 4
                }
#undef PTY_P4S
                if (bad) {
                    if (tl_s == 0) atomicOr(sl.status, bad);
                    if (local && tid == 0) s_dead[s] = 1;     // every CTA of the slot sees the same maxima
                    continue;
                }
                if (tl_s == 0) peak_part[((size_t)((step + 1) & 1) * P.nslots + s) * nq + rq] = npk;
                }
            }
        } else if constexpr (!BAT)                            // the batched flavour runs staged only
        for (int task = vcta * NTEAM + team; task < S * nq; task += ncta * NTEAM) {
            const int s = s0 + task / nq, rq = task % nq;
            if (s_dead[s] | (s_k[s] < 0)) continue;
            const SlotDev& sl = P.slot[s];
            const int j = s_j[s];
            const T* pkp = peak_part + ((size_t)(step & 1) * P.nslots + s) * nq;
            const T* omp = omax_part + ((size_t)(step & 1) * P.nslots + s) * nq;
            T peak = T(0), omax = T(0);
#pragma unroll
            for (int q = b; q < nq; q += B) {
                peak = fmax(peak, pkp[q]);
                omax = fmax(omax, omp[q]);
            }
            peak = group_max<B>(peak);
            omax = group_max<B>(omax);
            if (peak == T(0) || (P.update_probe && omax == T(0))) {   // engine.py:132-134, 145-147
                if (tl == 0) atomicOr(sl.status, peak == T(0) ? PTY_ERR_PROBE_ZERO : PTY_ERR_OBJECT_ZERO);
                if (local && tid == 0) s_dead[s] = 1;
                continue;
            }
            C* stg = P.sense == PTY_SENSE_XCORR_A ? reinterpret_cast<C*>(sl.stage) + (size_t)j * 2 * WW : nullptr;
            const T npk = task_row_inv_update<T, W>(tw, lines, numer, ppacc, nppacc, red4_p4, team, tl, gi, b, gmask,
                                                    scratch + (size_t)s * M * WW, M, rq, reinterpret_cast<C*>(sl.obj),
                                                    reinterpret_cast<T*>(P.ppg) + (size_t)s * WW,
                                                    sl.Wc, s_ar[s], s_ac[s], reinterpret_cast<C*>(sl.probes), peak,
                                                    omax, U, stg);
            if (tl == 0) peak_part[((size_t)((step + 1) & 1) * P.nslots + s) * nq + rq] = npk;
        }
        stamp(step, 7);
        if constexpr (!BAT) phase_sync();
        stamp(step, 8);
        if (P.timeline && step == 0 && tid == 0) {      // debug: the CTA's SM id replaces stamp (0, 8)
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            P.timeline[(size_t)8 * gridDim.x + blockIdx.x] = sm;
        }
        if (P.timeline && step == 1 && tid == 0 && P.timeline_steps > 1)   // ... and the virtual CTA index stamp (1, 8)
            P.timeline[(size_t)17 * gridDim.x + blockIdx.x] = (unsigned long long)vcta;
    }
}

// Deterministic end-of-sweep reduction of the per-visit error partials
// (engine.py:198-202, 239-241) in two fixed-order levels: one CTA per visit
// reduces its nCT column partials, then one CTA per slot reduces the visits.
struct ErrOut {
    double* p[kMaxSlots];
};
static __global__ void __launch_bounds__(256) err_visit_kernel(const double* err_part, int nCT, double* visit_sum) {
    __shared__ double red[32];
    const size_t v = blockIdx.x;
    double num = 0.0, den = 0.0, worst = 0.0;
    for (int ct = threadIdx.x; ct < nCT; ct += blockDim.x) {
        const double* e = err_part + (v * nCT + ct) * 3;
        num += e[0];
        den += e[1];
        worst = fmax(worst, e[2]);
    }
    num = block_sum(num, red);
    den = block_sum(den, red);
    worst = block_max(worst, red);
    if (threadIdx.x == 0) {
        visit_sum[v * 3] = num;
        visit_sum[v * 3 + 1] = den;
        visit_sum[v * 3 + 2] = worst;
    }
}
static __global__ void __launch_bounds__(256) err_slot_kernel(const double* visit_sum, int N, int nslots, ErrOut outs) {
    __shared__ double red[32];
    const int s = blockIdx.x;
    if (s >= nslots) return;
    double num = 0.0, den = 0.0, worst = 0.0;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const double* e = visit_sum + ((size_t)s * N + k) * 3;
        num += e[0];
        den += e[1];
        worst = fmax(worst, e[2]);
    }
    num = block_sum(num, red);
    den = block_sum(den, red);
    worst = block_max(worst, red);
    if (threadIdx.x == 0) {
        outs.p[s][0] = num;
        outs.p[s][1] = den;
        outs.p[s][2] = worst;
    }
}

}  // namespace pty
