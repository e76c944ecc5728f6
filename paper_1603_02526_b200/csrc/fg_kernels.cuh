// Kernels of the B200 factor-graph ADMM engine.
//
// One ADMM iteration (engine.py:483-516) runs as:
//   edge pass   : one kernel per (kind, slot dims) group.  Reads u and z,
//                 forms n = z[zmap] - u (phase n of the previous iteration,
//                 engine.py:292-298), applies the kind's prox (phase x,
//                 engine.py:257-261), writes x.
//   variable pass: per z component, m = x + u (phase m, engine.py:263-265),
//                 the exact NumPy reduceat tree of m*rho (phase z,
//                 engine.py:267-280), z = sum / z_weights, then
//                 u += alpha (x - z) (phase u, engine.py:282-290) and the
//                 residual partial sums (engine.py:398-406).  u is
//                 ping-ponged so the previous u survives for m.
//   reduce      : residuals, tolerance stop, iteration counter.
#pragma once

#include "fg_device.cuh"
#include "fg_edge.cuh"

namespace fg {

// ===========================================================================
// Variable pass
// ===========================================================================
enum { MODE_FUSED = 0, MODE_PHASEZ = 1 };

struct PassB {
    VarTab vt;
    const double* x;
    const double* uin;
    double* uout;
    const double* msrc;      // PHASEZ: materialized m
    double* z;               // z written by this pass
    const double* zin;       // z of the previous iteration (== z in PHASEZ)
    const double* rho;
    const double* alpha;
    const double* zw;
    Ctrl* ctrl;
    double* part;            // residual partials, 2 per slot
    const int32_t* zvar;     // z component -> variable
};

struct CompRef {
    int64_t pb;              // payload base of the variable
    int32_t eb, deg, d, c;   // edge base, degree, dim, component
};

__device__ __forceinline__ CompRef comp_ref(const PassB& b, int32_t k) {
    const int32_t v = b.zvar[k];
    CompRef r;
    r.pb = b.vt.pbase[v];
    r.eb = b.vt.ebase[v];
    r.deg = b.vt.deg[v];
    r.d = b.vt.dim[v];
    r.c = (int32_t)(k - b.vt.zbase[v]);
    return r;
}

// UNIT: every edge weight is exactly 1.0 (checked at sync), so m * rho is
// m and the rho stream is not read.
template <int MODE, bool UNIT = false>
struct ValFn {
    const double* x;
    const double* u;         // FUSED: u_in;  PHASEZ: materialized m
    const double* rho;
    CompRef r;
    bool* badm;
    __device__ __forceinline__ ValFn(const PassB& b, const CompRef& rr, bool* bm)
        : x(b.x), u(MODE == MODE_FUSED ? b.uin : b.msrc), rho(b.rho), r(rr),
          badm(bm) {}
    __device__ __forceinline__ double operator()(int64_t e) const {
        const int64_t p = r.pb + e * r.d + r.c;
        double m;
        if (MODE == MODE_FUSED) {
            m = x[p] + u[p];                         // phase m
            *badm |= !finite(m);
        } else {
            m = u[p];
        }
        if (UNIT) return m;
        return m * rho[r.eb + e];                    // engine.py:278
    }
    // the same value split into its loads and its arithmetic, so a caller
    // can issue many elements' loads before any of them is used
    struct Raw { double x, u, w; };
    __device__ __forceinline__ Raw load(int64_t e) const {
        const int64_t p = r.pb + e * r.d + r.c;
        Raw v;
        v.x = MODE == MODE_FUSED ? x[p] : 0.0;
        v.u = u[p];
        v.w = UNIT ? 1.0 : rho[r.eb + e];
        return v;
    }
    __device__ __forceinline__ double value(const Raw& v) const {
        double m;
        if (MODE == MODE_FUSED) {
            m = v.x + v.u;
            *badm |= !finite(m);
        } else {
            m = v.u;
        }
        if (UNIT) return m;
        return m * v.w;
    }
};

// u update + residual partials for elements [e0, e1) of one component.
// UNIT: rho = alpha = 1 exactly (rd = dz, t * alpha = t), not read.
template <bool UNIT = false, int NB = 4>
__device__ __forceinline__ void update_range(const PassB& b, const CompRef& r,
                                             int64_t e0, int64_t e1,
                                             int64_t step, double zn, double zo,
                                             double& pp, double& dd, bool& badu) {
    const double dz = zn - zo;
    // batches of NB elements: all loads before the stores (the compiler
    // cannot prove uout aliases nothing read here), one round trip each
    for (int64_t e = e0; e < e1; e += NB * step) {
        double xv[NB], uv[NB], rv[NB], av[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int64_t ee = e + k * step;
            if (ee < e1) {
                const int64_t p = r.pb + ee * r.d + r.c;
                xv[k] = b.x[p];
                uv[k] = b.uin[p];
                if (!UNIT) {
                    rv[k] = b.rho[r.eb + ee];
                    av[k] = b.alpha[r.eb + ee];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int64_t ee = e + k * step;
            if (ee < e1) {
                const double t = xv[k] - zn;             // engine.py:288
                pp += t * t;                             // engine.py:402
                const double rd = UNIT ? dz : rv[k] * dz;            // engine.py:403-405
                dd += rd * rd;
                const double un = UNIT ? uv[k] + t : uv[k] + t * av[k];     // :289-290
                b.uout[r.pb + ee * r.d + r.c] = un;
                badu |= !finite(un);
            }
        }
    }
}

// Tree program layout (int32): [nu, nlev, units(2*nu: start,len),
// level_cnt(nlev), ops(2*(nu-1): a,b)].  Node ids: units 0..nu-1, then
// internal nodes in level order; the root is the last node.
constexpr int kVarThreads = 256;
constexpr int kMaxUnits = 160;          // chunk <= 8192 -> <= 128 leaves

template <class F, int NT = kVarThreads, bool BATCH = false>
__device__ __forceinline__ double run_units_and_tree(F val, int64_t base_elem,
                                                     const int32_t* P,
                                                     double* sv) {
    const int nu = P[0], nlev = P[1];
    const int32_t* units = P + 2;
    const int32_t* lev = units + 2 * nu;
    const int32_t* ops = lev + nlev;
    // the top's level counts and operand ids, staged while the leaves load
    // (the level loop then waits on no global memory)
    __shared__ int32_t s_prog[2 * kMaxUnits + 64];
    const int nops = 2 * (nu - 1);
    for (int i = threadIdx.x; i < nops + nlev; i += NT) s_prog[i] = i < nops ? ops[i] : lev[i - nops];
    const int g = threadIdx.x >> 3, j = threadIdx.x & 7;
    constexpr int NG = NT / 8;
    for (int r0 = 0; r0 < nu; r0 += NG) {
        const int L = r0 + g;
        int64_t s = 0, len = 0;
        if (L < nu) { s = units[2 * L]; len = units[2 * L + 1]; }
        const double res = BATCH ? leaf_group8_batched(val, base_elem + s, len, j)
                                 : leaf_group8(val, base_elem + s, len, j);
        if (L < nu && j == 0) sv[L] = res;
    }
    __syncthreads();
    int node = nu, op = 0;
    for (int l = 0; l < nlev; ++l) {
        const int cnt = s_prog[nops + l];
        for (int o = threadIdx.x; o < cnt; o += NT)
            sv[node + o] = sv[s_prog[2 * (op + o)]] + sv[s_prog[2 * (op + o) + 1]];
        __syncthreads();
        node += cnt;
        op += cnt;
    }
    return sv[node - 1];
}

// Class L: 32 < degree <= chunk+1.  One CTA per z component: leaves by
// 8-lane groups, level-ordered combine in shared memory, then z and the
// u update of the whole segment.
template <int MODE>
__global__ void __launch_bounds__(kVarThreads) k_var_large(
    PassB b, const int32_t* list, const int32_t* progoff, const int32_t* prog,
    int64_t part_off) {
    __shared__ double sv[2 * kMaxUnits];
    __shared__ double sm[16];
    __shared__ double s_z[2];
    __shared__ int s_stop;
    if (threadIdx.x == 0) s_stop = b.ctrl->stop;
    __syncthreads();
    if (s_stop) return;
    const int64_t it = b.ctrl->iter;
    const int32_t k = list[blockIdx.x];
    const CompRef r = comp_ref(b, k);
    bool bm = false, bz = false, bu = false;
    ValFn<MODE> val(b, r, &bm);
    const double T = run_units_and_tree(val, 1, prog + progoff[blockIdx.x], sv);
    if (threadIdx.x == 0) {
        const double zn = ddiv(val(0) + T, b.zw[k]);
        bz = !finite(zn);
        s_z[0] = zn;
        s_z[1] = (MODE == MODE_FUSED) ? b.zin[k] : 0.0;
        b.z[k] = zn;
    }
    __syncthreads();
    double pp = 0.0, dd = 0.0;
    if (MODE == MODE_FUSED) {
        update_range(b, r, threadIdx.x, r.deg, kVarThreads, s_z[0], s_z[1], pp, dd, bu);
        if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
        if (bz) flag_error(b.ctrl, it, FG_PHASE_Z, false);
        if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
        block_sum2<kVarThreads>(pp, dd, sm);
        if (threadIdx.x == 0) {
            b.part[2 * (part_off + blockIdx.x)] = pp;
            b.part[2 * (part_off + blockIdx.x) + 1] = dd;
        }
    }
}

// Class G (degree > chunk+1), three kernels.
// G1: one CTA per chunk (a maximal pairwise subtree of <= chunk items).
struct GChunk { int32_t gi, start, progoff, pad; };
// G2 descriptor: top program offset, first chunk, cut slot (or -1)
struct GComp { int32_t topoff, cbase, pad0, pad1; };
__device__ __forceinline__ int32_t comps_topoff(const GComp* c, int gi) { return c[gi].topoff; }
template <int MODE, int NT = kVarThreads>
__device__ void giant_top_body(const PassB& b, const int32_t* glist, const GComp* comps,
                               const int32_t* prog, const double* csum, double* gz,
                               double* send, int gi, double* sv, int64_t it,
                               const CompRef* known = nullptr);
// With `comps` non-null the last CTA to finish a component's chunks (an
// atomic counter per component, reset by that CTA) also evaluates the top
// of its tree: the separate top launch disappears.  The top program is the
// same whichever CTA runs it, so the result is deterministic.
template <int MODE, int NT = kVarThreads, bool UNIT = false>
__global__ void __launch_bounds__(NT) k_var_giant_chunks(
    PassB b, const int32_t* glist, const GChunk* chunks, const int32_t* prog,
    double* csum, const GComp* comps = nullptr, double* gz = nullptr, double* send = nullptr,
    unsigned* counters = nullptr, const CompRef* cref = nullptr) {
    extern __shared__ double sv_top[];
    __shared__ int s_last;
    __shared__ double sv[2 * kMaxUnits];
    __shared__ int s_stop;
    if (threadIdx.x == 0) s_stop = b.ctrl->stop;
    __syncthreads();
    if (s_stop) return;
    const int64_t it = b.ctrl->iter;
    const GChunk ch = chunks[blockIdx.x];
    // the per-chunk table loads with the descriptor (no dependent chain
    // glist -> zvar -> variable table before the leaf loads)
    const CompRef r = cref ? cref[blockIdx.x] : comp_ref(b, glist[ch.gi]);
    bool bm = false;
    ValFn<MODE, UNIT> val(b, r, &bm);
    // pad = first element of the tree: 1 for a whole segment (a[0] is the
    // reduceat initial value), 0 for a rank's local part of a cut segment
    const double T = run_units_and_tree<ValFn<MODE, UNIT>, NT, true>(val, (int64_t)ch.pad + ch.start,
                                                         prog + ch.progoff, sv);
    if (threadIdx.x == 0) csum[blockIdx.x] = T;
    if (MODE == MODE_FUSED && bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (comps) {
        if (threadIdx.x == 0) {
            __threadfence();
            const int nu = prog[comps_topoff(comps, ch.gi)];
            s_last = atomicAdd(counters + ch.gi, 1u) == (unsigned)(nu - 1);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            giant_top_body<MODE, NT>(b, glist, comps, prog, csum, gz, send, ch.gi, sv_top, it, &r);
            if (threadIdx.x == 0) counters[ch.gi] = 0u;
        }
    }
}

// G2 (run by the last chunk CTA of each component): combine chunk sums
// along the top of the tree (program whose units are chunks), then z.  A
// cut component (pad0 = its position in the exchange vector) instead
// stores its local partial sum in `send`; z follows after the exchange
// (k_cut_finalize).
// Top of giant component gi's tree from its chunk sums -> z (or the cut
// partial); one CTA, `sv` holds 2 doubles per chunk.
template <int MODE, int NT>
__device__ void giant_top_body(const PassB& b, const int32_t* glist, const GComp* comps,
                               const int32_t* prog, const double* csum, double* gz,
                               double* send, int gi, double* sv, int64_t it,
                               const CompRef* known) {
    const GComp gc = comps[gi];
    const int32_t k = glist[gi];
    const int32_t* P = prog + gc.topoff;
    const int nu = P[0], nlev = P[1];
    const int32_t* lev = P + 2 + 2 * nu;
    const int32_t* ops = lev + nlev;
    // one round trip: chunk sums, the top program (into shared memory after
    // the 2 nu node values) and, on thread 0, element 0 and the z inputs
    int32_t* s_prog = reinterpret_cast<int32_t*>(sv + 2 * nu);
    const int nops = nu > 0 ? 2 * (nu - 1) : 0;
    for (int u = threadIdx.x; u < nu; u += NT) sv[u] = __ldcg(csum + gc.cbase + u);
    for (int i = threadIdx.x; i < nops + nlev; i += NT) s_prog[i] = i < nops ? ops[i] : lev[i - nops];
    double a0 = 0.0, zw = 1.0, zo = 0.0;
    bool bm = false;
    if (threadIdx.x == 0 && gc.pad0 < 0) {
        const CompRef r = known ? *known : comp_ref(b, k);
        ValFn<MODE> val(b, r, &bm);
        a0 = val(0);
        zw = b.zw[k];
        zo = (MODE == MODE_FUSED) ? b.zin[k] : 0.0;
    }
    __syncthreads();
    int node = nu, op = 0;
    for (int l = 0; l < nlev; ++l) {
        const int cnt = s_prog[nops + l];
        for (int o = threadIdx.x; o < cnt; o += NT)
            sv[node + o] = sv[s_prog[2 * (op + o)]] + sv[s_prog[2 * (op + o) + 1]];
        __syncthreads();
        node += cnt;
        op += cnt;
    }
    if (gc.pad0 >= 0) {
        if (threadIdx.x == 0) send[gc.pad0] = (nu > 0) ? sv[node - 1] : 0.0;
        return;
    }
    if (threadIdx.x == 0) {
        const double zn = ddiv(a0 + sv[node - 1], zw);
        gz[2 * gi] = zn;
        gz[2 * gi + 1] = zo;
        b.z[k] = zn;
        if (MODE == MODE_FUSED) {
            if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
            if (!finite(zn)) flag_error(b.ctrl, it, FG_PHASE_Z, false);
        }
    }
}

// Residuals, tolerance stop and iteration bookkeeping (engine.py:502-516)
// over partial slots [0, npart) minus [skip_lo, skip_hi), by one CTA of NT
// threads.
// The control fields the commit reads, loaded by thread 0 BEFORE the
// partial sums so their round trip overlaps the partials' loads.
struct CtrlIn {
    int64_t it;
    double scale, ptol, dtol;
    bool err;
};
__device__ __forceinline__ CtrlIn ctrl_in(const Ctrl* c) {
    CtrlIn r;
    r.it = c->iter;
    r.scale = c->scale;
    r.ptol = c->primal_tol;
    r.dtol = c->dual_tol;
    r.err = c->err_key != ~0ull;
    return r;
}

// Thread 0's part of the reduction: residual norms, history row,
// completion, stop decision and the iteration counter from the two summed
// partials.
__device__ __forceinline__ void reduce_commit(Ctrl* c, const CtrlIn& in, double a, double bsum,
                                              double* hist) {
    const int64_t it = in.it;
    const double primal = sqrt(a) * in.scale;
    const double dual = sqrt(bsum) * in.scale;
    c->primal = primal;
    c->dual = dual;
    if (hist) { hist[2 * (it - 1)] = primal; hist[2 * (it - 1) + 1] = dual; }
    c->completed = it;
    if (in.err) {
        c->stop = 1;
    } else {
        const bool pc = in.ptol > 0.0, dc = in.dtol > 0.0;
        bool ok = pc || dc;
        if (pc) ok = ok && (primal <= in.ptol);
        if (dc) ok = ok && (dual <= in.dtol);
        if (ok) { c->converged = 1; c->stop = 1; }
    }
    c->iter = it + 1;
}

// Residuals, tolerance stop and iteration bookkeeping (engine.py:502-516)
// over partial slots [0, npart) minus [skip_lo, skip_hi), by one CTA of NT
// threads.  Each thread sums its slots in index order (loads unrolled by
// 4, additions in the same order), then the fixed block tree.
template <int NT>
__device__ void reduce_body(Ctrl* c, const double* part, int64_t npart, double* hist,
                            int64_t skip_lo, int64_t skip_hi, double* sm) {
    CtrlIn in{};
    if (threadIdx.x == 0) in = ctrl_in(c);
    double a = 0.0, bsum = 0.0;
    // slots i = tid, tid + NT, ... below `hi`, loads 4 at a time
    auto range = [&](int64_t i, int64_t hi) {
        for (; i + 3 * NT < hi; i += 4 * NT) {
            double v[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[2 * k] = __ldcg(part + 2 * (i + k * NT));
                v[2 * k + 1] = __ldcg(part + 2 * (i + k * NT) + 1);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                a += v[2 * k];
                bsum += v[2 * k + 1];
            }
        }
        for (; i < hi; i += NT) {
            a += __ldcg(part + 2 * i);
            bsum += __ldcg(part + 2 * i + 1);
        }
        return i;
    };
    int64_t i = threadIdx.x;
    if (skip_hi > skip_lo) {
        i = range(i, skip_lo < npart ? skip_lo : npart);
        if (i < skip_hi) i += (skip_hi - i + NT - 1) / NT * NT;   // same progression
    }
    range(i, npart);
    block_sum2<NT>(a, bsum, sm);
    if (threadIdx.x == 0) reduce_commit(c, in, a, bsum, hist);
}

// Optional fused reduction: the last CTA of the update runs reduce_body
// (when the update is the iteration's last variable kernel).
struct FusedReduce {
    unsigned* counter;             // null: no fused reduction
    int64_t npart, skip_lo, skip_hi;
    double* hist;
};

// G3: u update of giant components, one CTA per element range.
struct GWork { int32_t gi, e0, e1, pad; };
template <bool UNIT = false>
__global__ void __launch_bounds__(kVarThreads, UNIT ? 4 : 2) k_var_giant_update(
    PassB b, const int32_t* glist, const GWork* work, const double* gz,
    int64_t part_off, FusedReduce fr = FusedReduce{nullptr, 0, 0, 0, nullptr},
    const CompRef* wref = nullptr) {
    __shared__ double sm[16];
    __shared__ int s_last;
    __shared__ int s_stop;
    if (threadIdx.x == 0) s_stop = b.ctrl->stop;
    __syncthreads();
    if (s_stop) return;
    const int64_t it = b.ctrl->iter;
    const GWork wk = work[blockIdx.x];
    const CompRef r = wref ? wref[blockIdx.x] : comp_ref(b, glist[wk.gi]);
    double pp = 0.0, dd = 0.0;
    bool bu = false;
    update_range<UNIT, 4>(b, r, wk.e0 + threadIdx.x, wk.e1, kVarThreads, gz[2 * wk.gi],
                          gz[2 * wk.gi + 1], pp, dd, bu);
    if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kVarThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
    if (fr.counter) {
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(fr.counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            reduce_body<kVarThreads>(b.ctrl, b.part, fr.npart, fr.hist, fr.skip_lo, fr.skip_hi, sm);
            if (threadIdx.x == 0) *fr.counter = 0u;
        }
    }
}

// Residuals, tolerance stop and iteration bookkeeping (engine.py:502-516).
// Partial slots [skip_lo, skip_hi) are not written by this iteration's
// kernels (the fused chain uses fewer slots than the classes it replaces).
__global__ void __launch_bounds__(1024) k_reduce(Ctrl* c, const double* part,
                                                 int64_t npart, double* hist,
                                                 int64_t skip_lo = 0, int64_t skip_hi = 0) {
    __shared__ double sm[64];
    __shared__ int s_stop;
    if (threadIdx.x == 0) s_stop = c->stop;
    __syncthreads();
    if (s_stop) return;
    reduce_body<1024>(c, part, npart, hist, skip_lo, skip_hi, sm);
}

// Cut components after the exchange: rank-order sum of the all-gathered
// partials (identical on every rank), then z as for a whole segment.
__device__ __forceinline__ void cut_finalize_one(const PassB& b, const int32_t* glist,
                                                 const GComp* comps, const int32_t* cutg,
                                                 int64_t t, const double* recv, int32_t world,
                                                 int64_t ncut, double* gz) {
    const int32_t gi = cutg[t];
    const GComp gc = comps[gi];
    const int32_t k = glist[gi];
    double tot = recv[gc.pad0];
    for (int r = 1; r < world; ++r) tot = tot + recv[(int64_t)r * ncut + gc.pad0];
    const double zn = ddiv(tot, b.zw[k]);
    gz[2 * gi] = zn;
    gz[2 * gi + 1] = b.zin[k];
    b.z[k] = zn;
    if (!finite(zn)) flag_error(b.ctrl, b.ctrl->iter, FG_PHASE_Z, false);
}

__global__ void k_cut_finalize(PassB b, const int32_t* glist, const GComp* comps,
                               const int32_t* cutg, int64_t ncutg,
                               const double* recv, int32_t world, int64_t ncut,
                               double* gz) {
    if (b.ctrl->stop == 1) return;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncutg) return;
    cut_finalize_one(b, glist, comps, cutg, t, recv, world, ncut, gz);
}

// Partitioned runs split the residual reduction: local sums (plus the local
// error key) go to a 4-double send slot, are all-gathered, and every rank
// combines them in rank order, so all ranks take the same stop decision.
// this rank's residual partial sums and error key -> send4[0..3]; one CTA
// of NT threads
template <int NT>
__device__ __forceinline__ void reduce_local_body(const Ctrl* c, const double* part,
                                                  int64_t npart, double* send4,
                                                  int64_t skip_lo, int64_t skip_hi,
                                                  double* sm) {
    double a = 0.0, bsum = 0.0;
    for (int64_t i = threadIdx.x; i < npart; i += NT) {
        if (i >= skip_lo && i < skip_hi) continue;
        a += part[2 * i];
        bsum += part[2 * i + 1];
    }
    block_sum2<NT>(a, bsum, sm);
    if (threadIdx.x == 0) {
        send4[0] = a;
        send4[1] = bsum;
        send4[2] = __longlong_as_double((long long)c->err_key);
        send4[3] = 0.0;
    }
}

__global__ void __launch_bounds__(1024) k_reduce_local(Ctrl* c, const double* part,
                                                       int64_t npart, double* send4,
                                                       int64_t skip_lo = 0, int64_t skip_hi = 0) {
    __shared__ double sm[64];
    reduce_local_body<1024>(c, part, npart, send4, skip_lo, skip_hi, sm);
}

// Rank-order combination of the all-gathered 4-double slots (thread 0):
// residual norms, history row, error key, stop decision.
__device__ __forceinline__ void reduce_final_commit(Ctrl* c, const double* recv4, int32_t world,
                                                    double* hist) {
    if (c->stop == 1) return;
    double a = recv4[0], bsum = recv4[1];
    unsigned long long err = (unsigned long long)__double_as_longlong(recv4[2]);
    for (int r = 1; r < world; ++r) {
        a = a + recv4[4 * r];
        bsum = bsum + recv4[4 * r + 1];
        const unsigned long long e = (unsigned long long)__double_as_longlong(recv4[4 * r + 2]);
        err = e < err ? e : err;
    }
    const int64_t it = c->iter;
    const double primal = sqrt(a) * c->scale;
    const double dual = sqrt(bsum) * c->scale;
    c->primal = primal;
    c->dual = dual;
    if (hist) { hist[2 * (it - 1)] = primal; hist[2 * (it - 1) + 1] = dual; }
    if (err != ~0ull) {
        if (err < c->err_key) c->err_key = err;
        c->stop = 1;
        c->completed = it - 1;
        return;
    }
    c->completed = it;
    const bool pc = c->primal_tol > 0.0, dc = c->dual_tol > 0.0;
    bool ok = pc || dc;
    if (pc) ok = ok && (primal <= c->primal_tol);
    if (dc) ok = ok && (dual <= c->dual_tol);
    if (ok) { c->converged = 1; c->stop = 1; }
    c->iter = it + 1;
}

__global__ void k_reduce_final(Ctrl* c, const double* recv4, int32_t world,
                               double* hist) {
    if (threadIdx.x != 0) return;
    reduce_final_commit(c, recv4, world, hist);
}

// ===========================================================================
// Layout conversion, unfused phases, host-API residuals
// ===========================================================================

// dst[p] = src_ref[vm2ref[p]]      (reference order -> var-major)
__global__ void k_gather_from_ref(int64_t P, const int64_t* vm2ref,
                                  const double* src_ref, double* dst) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P) dst[p] = src_ref[vm2ref[p]];
}

// dst_ref[vm2ref[p]] = f(p):  0 x, 1 x + uprev (m), 2 ucur, 3 z - ucur (n)
__global__ void k_scatter_to_ref(int64_t P, const int64_t* vm2ref,
                                 const int32_t* vmz, int mode, const double* x,
                                 const double* ucur, const double* uprev,
                                 const double* z, double* dst_ref,
                                 unsigned long long* first_bad) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    double v;
    if (mode == 0) v = x[p];
    else if (mode == 1) v = x[p] + uprev[p];
    else if (mode == 2) v = ucur[p];
    else v = z[vmz[p]] - ucur[p];
    const int64_t r = vm2ref[p];
    dst_ref[r] = v;
    // first non-finite entry in reference order (the host reports it
    // without scanning the downloaded array)
    if (!isfinite(v)) atomicMin(first_bad, (unsigned long long)r);
}

// edge-indexed gather: dst[q] = src_ref[ref_edge[q]]
__global__ void k_gather_edges(int64_t E, const int32_t* ref_edge,
                               const double* src_ref, double* dst) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < E) dst[q] = src_ref[ref_edge[q]];
}

// phase m (engine.py:263-265): m = x + u
// Unit-weight checks (parameter sync).
// Per class-L row (one CTA each): its single non-unit edge, if any; a row
// with two or more raises the flag (the rows then keep the general form).
struct LExc { int32_t rank, pad; double rho, alpha; };
__global__ void k_unit_rows(const int32_t* vlist, VarTab vt, const double* rho,
                            const double* alpha, LExc* out, int32_t* flag) {
    __shared__ int s_cnt, s_rank;
    if (threadIdx.x == 0) { s_cnt = 0; s_rank = -1; }
    __syncthreads();
    const int32_t v = vlist[blockIdx.x];
    const int32_t e0 = vt.ebase[v], dg = vt.deg[v];
    for (int32_t k = threadIdx.x; k < dg; k += blockDim.x)
        if (rho[e0 + k] != 1.0 || alpha[e0 + k] != 1.0) {
            atomicAdd(&s_cnt, 1);
            atomicMax(&s_rank, k);         // read only when it is the single one
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        LExc o{-1, 0, 1.0, 1.0};
        if (s_cnt == 1) o = LExc{s_rank, 0, rho[e0 + s_rank], alpha[e0 + s_rank]};
        if (s_cnt > 1) atomicOr(flag, 1);
        out[blockIdx.x] = o;
    }
}

// ... and any collision edge (rows of the all-pairs triangle).
__global__ void k_unit_collision(GroupDev g, const double* rho, int32_t* flag) {
    const int i = blockIdx.x;
    if (i >= g.ndisks) return;
    const DiskRow R = disk_row(g, i);
    bool bad = false;
    for (int e = threadIdx.x; e < g.ndisks - 1; e += blockDim.x)
        bad |= rho[R.ebc + e] != 1.0 || rho[R.ebr + e] != 1.0;
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Any payload slot whose uploaded n differs (bitwise) from z[zmap] - u.
__global__ void k_n_mismatch(int64_t P, const int32_t* vmz, const double* z,
                             const double* u, const double* n, int32_t* flag) {
    bool bad = false;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P;
         q += (int64_t)gridDim.x * blockDim.x)
        bad |= __double_as_longlong(z[vmz[q]] - u[q]) != __double_as_longlong(n[q]);
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// The same test on the upload staging buffers (reference order), so it can
// run concurrently with iterations that overwrite the var-major state.
__global__ void k_n_check_ref(int64_t P, const int64_t* vm2ref, const int32_t* vmz,
                              const double* z, const double* u_ref, const double* n_ref,
                              int32_t* flag) {
    bool bad = false;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = vm2ref[q];
        bad |= __double_as_longlong(z[vmz[q]] - u_ref[r]) != __double_as_longlong(n_ref[r]);
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void k_phase_m(int64_t P, const double* x, const double* u, double* m) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P) m[p] = x[p] + u[p];
}

// phase n (engine.py:292-298): n = z[zmap] - u
__global__ void k_phase_n(int64_t P, const int32_t* vmz, const double* z,
                          const double* u, double* n) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P) n[p] = z[vmz[p]] - u[p];
}

// phase u (engine.py:282-290) one thread per var-major edge
__global__ void k_phase_u(int64_t E, VarTab vt, const int32_t* vm_var,
                          const double* x, const double* z,
                          const double* alpha, double* u) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= E) return;
    const int32_t v = vm_var[q];
    const int d = vt.dim[v];
    const int64_t p0 = vt.pbase[v] + (q - vt.ebase[v]) * (int64_t)d;
    const int64_t z0 = vt.zbase[v];
    const double al = alpha[q];
    for (int c = 0; c < d; ++c) u[p0 + c] = u[p0 + c] + (x[p0 + c] - z[z0 + c]) * al;
}

// ---- phase-profile kernels (RunConfig(profile=True)) -----------------------
// The five phases as separate launches, as the reference times them
// (engine.py:489-500), each with its non-finite check (engine.py:333-350)
// keyed by (iteration, phase) on the device.  Same arithmetic as the
// per-phase API kernels above; u is written to the other ping-pong slot so
// the previous u survives (m = x + u_prev at download).
__global__ void __launch_bounds__(256) k_prof_m(int64_t P, const double* x, const double* u,
                                                double* m, Ctrl* c) {
    if (c->stop) return;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    if (p < P) {
        const double v = x[p] + u[p];          // engine.py:263-265
        m[p] = v;
        bad = !finite(v);
    }
    if (bad) flag_error(c, c->iter, FG_PHASE_M, true);
}

// z check of the profile run (the phase-z kernels do not check in
// MODE_PHASEZ); outside the phase timers, as _check_finite is
__global__ void __launch_bounds__(256) k_prof_check_z(int64_t Z, const double* z, Ctrl* c) {
    if (c->stop) return;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < Z && !finite(z[k])) flag_error(c, c->iter, FG_PHASE_Z, true);
}

__global__ void __launch_bounds__(256) k_prof_u(int64_t E, VarTab vt, const int32_t* vm_var,
                                                const double* x, const double* z,
                                                const double* alpha, const double* uin,
                                                double* uout, Ctrl* c) {
    if (c->stop) return;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= E) return;
    const int32_t v = vm_var[q];
    const int d = vt.dim[v];
    const int64_t p0 = vt.pbase[v] + (q - vt.ebase[v]) * (int64_t)d;
    const int64_t z0 = vt.zbase[v];
    const double al = alpha[q];
    bool bad = false;
    for (int k = 0; k < d; ++k) {              // engine.py:282-290
        const double nu = uin[p0 + k] + (x[p0 + k] - z[z0 + k]) * al;
        uout[p0 + k] = nu;
        bad |= !finite(nu);
    }
    if (bad) flag_error(c, c->iter, FG_PHASE_U, true);
}

__global__ void __launch_bounds__(256) k_prof_n(int64_t P, const int32_t* vmz, const double* z,
                                                const double* u, double* n, Ctrl* c) {
    if (c->stop) return;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    if (p < P) {
        const double v = z[vmz[p]] - u[p];     // engine.py:292-298
        n[p] = v;
        bad = !finite(v);
    }
    if (bad) flag_error(c, c->iter, FG_PHASE_N, true);
}

// residuals (engine.py:398-406) on an explicit z_prev; per-block partials
__global__ void __launch_bounds__(256) k_residual_parts(
    int64_t E, VarTab vt, const int32_t* vm_var, const double* x,
    const double* z, const double* zprev, const double* rho, double* part) {
    __shared__ double sm[16];
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double pp = 0.0, dd = 0.0;
    if (q < E) {
        const int32_t v = vm_var[q];
        const int d = vt.dim[v];
        const int64_t p0 = vt.pbase[v] + (q - vt.ebase[v]) * (int64_t)d;
        const int64_t z0 = vt.zbase[v];
        for (int c = 0; c < d; ++c) {
            const double t = x[p0 + c] - z[z0 + c];
            pp += t * t;
            const double r = rho[q] * (z[z0 + c] - zprev[z0 + c]);
            dd += r * r;
        }
    }
    block_sum2<256>(pp, dd, sm);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = pp; part[2 * blockIdx.x + 1] = dd; }
}

__global__ void __launch_bounds__(1024) k_sum_parts(const double* part,
                                                    int64_t npart, double* out2) {
    __shared__ double sm[64];
    double a = 0.0, bsum = 0.0;
    for (int64_t i = threadIdx.x; i < npart; i += 1024) {
        a += part[2 * i];
        bsum += part[2 * i + 1];
    }
    block_sum2<1024>(a, bsum, sm);
    if (threadIdx.x == 0) { out2[0] = a; out2[1] = bsum; }
}

}  // namespace fg
