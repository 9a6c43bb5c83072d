// pty_batched_host.cuh -- host side of the batched extension: workspace
// layout, tile choice and the kernel sequence of pty_batch_contrib /
// pty_batch_apply.  Instantiated per (dtype, window) in pty_batch_*.cu.
#pragma once
#include "pty_batched.cuh"
#include "pty_host.cuh"

namespace pty {

struct BatchLayout {
    int* anchors;
    void *scratch, *onum, *pp, *pp_part, *omax_part, *tmax_part, *pgroup, *tile_max, *upd;
    size_t bytes;
};

struct BatchShape {
    int TR, TC, nRT, nCT, G, ntiles;
};

inline BatchShape batch_shape(int W, int M, int b, int H, int Wc) {
    BatchShape s;
    s.TR = 1;
    while (s.TR < W && s.TR * 2 * M <= 16) s.TR *= 2;         // <= 16 lines per row item
    s.TC = 4;                                                 // err_part is [N][W/4][3]
    s.nRT = W / s.TR;
    s.nCT = W / s.TC;
    const int want = 8 * sm_count();
    s.G = std::max(1, std::min(b, (want + s.nRT - 1) / s.nRT));
    s.ntiles = ((H + kObjTile - 1) / kObjTile) * ((Wc + kObjTile - 1) / kObjTile);
    return s;
}

template <typename T>
inline BatchLayout carve_batch(void* ws, int W, int M, int b, int H, int Wc, const BatchShape& sh, bool upd) {
    Carver c(ws);
    BatchLayout L{};
    const size_t WW = (size_t)W * W;
    L.anchors = c.take<int>((size_t)b * 2 * sizeof(int));
    L.scratch = c.take<void>((size_t)b * M * WW * sizeof(cplx<T>));
    L.onum = c.take<void>((size_t)b * WW * sizeof(cplx<T>));
    L.pp = c.take<void>(WW * sizeof(T));
    L.pp_part = c.take<void>((size_t)sh.nRT * sizeof(T));
    L.omax_part = c.take<void>((size_t)b * sh.nRT * sizeof(T));
    L.tmax_part = c.take<void>((size_t)b * sh.nCT * sizeof(T));
    L.pgroup = c.take<void>((size_t)sh.G * (2 * M + 1) * WW * sizeof(T));
    L.tile_max = c.take<void>((size_t)sh.ntiles * sizeof(T));
    L.upd = upd ? c.take<void>((size_t)H * Wc * sizeof(cplx<T>)) : nullptr;
    L.bytes = c.off;
    return L;
}

template <typename T, int W>
int fill_batch(const PtyBatchArgs* a, BatchDev& P, BatchShape& sh, cudaStream_t st) {
    const int M = a->modes, b = a->n_batch;
    sh = batch_shape(W, M, b, a->H, a->Wc);
    const bool upd = a->sense == PTY_SENSE_XCORR_A;
    BatchLayout L = carve_batch<T>(a->workspace, W, M, b, a->H, a->Wc, sh, upd);
    if (!a->workspace || a->workspace_bytes < (int64_t)L.bytes) return PTY_ERR_ARGUMENT;
    P = BatchDev{};
    P.W = W; P.M = M; P.N = a->n_positions; P.b = b;
    P.TR = sh.TR; P.TC = sh.TC; P.nRT = sh.nRT; P.nCT = sh.nCT; P.G = sh.G;
    P.lgTR = 0; while ((1 << P.lgTR) < sh.TR) ++P.lgTR;
    P.lgTC = 0; while ((1 << P.lgTC) < sh.TC) ++P.lgTC;
    P.obj = a->obj; P.H = a->H; P.Wc = a->Wc; P.r0 = a->r0; P.c0 = a->c0;
    P.probes = a->probes; P.patterns = a->patterns; P.positions = a->positions;
    P.batch = a->batch; P.visit0 = a->visit0;
    P.alpha_o = a->alpha_obj; P.alpha_p = a->alpha_probe; P.beta = a->beta; P.gamma = a->gamma;
    P.eps_rel = a->epsilon_rel;
    P.update_probe = a->update_probe; P.track_mod = a->track_modulus; P.sense = a->sense;
    P.stage = a->stage; P.obj_acc = a->obj_acc; P.probe_acc = a->probe_acc;
    P.err_part = a->err_part; P.status = a->status;
    P.anchors = L.anchors; P.scratch = L.scratch; P.onum = L.onum; P.pp = L.pp; P.pp_part = L.pp_part;
    P.omax_part = L.omax_part; P.tmax_part = L.tmax_part; P.pgroup = L.pgroup; P.tile_max = L.tile_max;
    P.upd = L.upd;
    P.twiddles = twiddles<T, W>(st);
    if (!P.twiddles) return PTY_ERR_CUDA;
    return PTY_OK;
}

template <typename K> inline int set_smem(K kern, size_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess
               ? PTY_OK : PTY_ERR_CUDA;
}

template <typename T, int W>
int run_batch_contrib(const PtyBatchArgs* a, cudaStream_t st) {
    BatchDev P;
    BatchShape sh;
    int rc = fill_batch<T, W>(a, P, sh, st);
    if (rc) return rc;
    const int M = a->modes, b = a->n_batch;
    constexpr int LS = line_stride<W>();
    const size_t fix = (size_t)W * sizeof(cplx<T>) + 64 * sizeof(double);
    const size_t s_rows = fix + (size_t)sh.TR * M * LS * sizeof(cplx<T>);
    const size_t s_cols = fix + (size_t)sh.TC * M * LS * sizeof(cplx<T>);
    const size_t s_inv = s_rows + (size_t)M * sh.TR * W * sizeof(cplx<T>) + (size_t)sh.TR * W * sizeof(T);
    const size_t s_gather = (size_t)b * sizeof(int);
    if (s_gather > max_dyn_smem()) return PTY_ERR_ARGUMENT;      // batch too large for one gather list
    if ((rc = set_smem(bk_rows_fwd<T, W>, s_rows)) || (rc = set_smem(bk_cols_fwd<T, W>, s_cols)) ||
        (rc = set_smem(bk_cols_mod<T, W>, s_cols)) || (rc = set_smem(bk_rows_inv<T, W>, s_inv)) ||
        (rc = set_smem(bk_obj_gather<T, W>, s_gather)))
        return rc;
    const size_t HW = (size_t)a->H * a->Wc, WW = (size_t)W * W;
    cudaMemsetAsync(a->obj_acc, 0, 3 * HW * sizeof(T), st);
    cudaMemsetAsync(a->probe_acc, 0, (size_t)(2 * M + 1) * WW * sizeof(T), st);
    bk_probe_power<T, W><<<std::max(sh.nRT, (b + kBatThreads - 1) / kBatThreads), kBatThreads, 0, st>>>(P);
    bk_rows_fwd<T, W><<<b * sh.nRT, kBatThreads, s_rows, st>>>(P);
    bk_cols_fwd<T, W><<<b * sh.nCT, kBatThreads, s_cols, st>>>(P);
    bk_cols_mod<T, W><<<b * sh.nCT, kBatThreads, s_cols, st>>>(P);
    bk_rows_inv<T, W><<<sh.nRT * sh.G, kBatThreads, s_inv, st>>>(P);
    bk_probe_reduce<T, W><<<std::min<size_t>(4096, ((2 * M + 1) * WW + 255) / 256), 256, 0, st>>>(P);
    bk_obj_gather<T, W><<<sh.ntiles, 256, s_gather, st>>>(P);
    count(7);
    return last_status();
}

template <typename T, int W>
int run_batch_apply(const PtyBatchArgs* a, cudaStream_t st) {
    BatchDev P;
    BatchShape sh;
    int rc = fill_batch<T, W>(a, P, sh, st);
    if (rc) return rc;
    const size_t HW = (size_t)a->H * a->Wc, WW = (size_t)W * W;
    bk_obj_tile_max<T, W><<<sh.ntiles, 256, 0, st>>>(P);
    bk_obj_apply<T, W><<<(unsigned)std::min<size_t>(8 * sm_count(), (HW + 255) / 256), 256, 0, st>>>(P, sh.ntiles);
    int n = 2;
    if (a->update_probe) {
        bk_probe_apply<T, W><<<(unsigned)std::min<size_t>(2 * sm_count(), (WW + 255) / 256), 256, 0, st>>>(P);
        ++n;
    }
    if (a->sense == PTY_SENSE_XCORR_A) {
        bk_stage_after<T, W><<<a->n_batch * sh.nRT, 256, 0, st>>>(P);
        ++n;
    }
    count(n);
    return last_status();
}

template <typename T, int W>
int64_t batch_workspace(int M, int b, int H, int Wc, bool upd) {
    BatchShape sh = batch_shape(W, M, b, H, Wc);
    return (int64_t)carve_batch<T>(nullptr, W, M, b, H, Wc, sh, upd).bytes;
}

}  // namespace pty
