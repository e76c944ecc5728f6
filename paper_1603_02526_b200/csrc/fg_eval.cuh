// Objective and constraint violation at a consensus vector z, on the device.
//
// Reference: FactorGraph.objective_value / constraint_violation
// (graph.py:253-263) sum each factor's `objective` and take the max of its
// `violation` (operators.py, per kind) over Python factor objects.  Here one
// thread evaluates one factor from z (slot offsets as in the edge pass),
// CTAs reduce (sum / max) into per-CTA partials, and the host combines
// them in CTA order.  Kinds without an objective or constraint contribute 0
// as in the reference's base class (prox.py:94-100).
#pragma once

#include "fg_edge.cuh"

namespace fg {

__device__ __forceinline__ double sq(double v) { return v * v; }

// per-factor (objective, violation) for each kind
__device__ void eval_factor(const GroupDev& g, const double* z, const VarTab& vt,
                            const FRef& r, double& obj, double& vio) {
    const double* P = g.fp ? g.fp + r.f * g.fstride : nullptr;
    obj = 0.0;
    vio = 0.0;
    auto zs = [&](int j) { return z + locate(vt, g, j, r).zo; };
    switch (g.kind) {
        case FG_KIND_QUADRATIC: {            // operators.py:137-141
            int off = 0;
            for (int j = 0; j < g.nslots; ++j) {
                const double* v = zs(j);
                const int d = g.dim[j];
                double s = 0.0;
                for (int c = 0; c < d; ++c) s += sq(v[c] - P[off + c]);
                obj += 0.5 * P[off + d] * s;
                off += d + 1;
            }
            break;
        }
        case FG_KIND_COLLISION: {            // operators.py:193-196
            const double* c1 = zs(0);
            const double* c2 = zs(2);
            const double gap = (zs(1)[0] + zs(3)[0]) -
                               sqrt(sq(c1[0] - c2[0]) + sq(c1[1] - c2[1]));
            vio = gap > 0.0 ? gap : 0.0;
            break;
        }
        case FG_KIND_WALL: {                 // operators.py:236-238, :39-41
            const double* c = zs(0);
            const double m = (P[0] * (c[0] - P[2]) + P[1] * (c[1] - P[3])) - zs(1)[0];
            vio = -m > 0.0 ? -m : 0.0;
            break;
        }
        case FG_KIND_RADIUS:                 // operators.py:279-280
            obj = -0.5 * P[0] * sq(zs(0)[0]);
            break;
        case FG_KIND_MPC_COST: {             // operators.py:316-319
            const double* v = zs(0);
            double s = 0.0;
            for (int c = 0; c < g.dim[0]; ++c) s += P[c] * v[c] * v[c];
            obj = 0.5 * s;
            break;
        }
        case FG_KIND_MPC_INIT: {             // operators.py:356-358
            const double* v = zs(0);
            for (int c = 0; c < g.fstride; ++c) vio = fmax(vio, fabs(v[c] - P[c]));
            break;
        }
        case FG_KIND_MPC_DYN: {              // operators.py:406-410
            const double* v0 = zs(0);
            const double* v1 = zs(1);
            const int d = g.ip, n0 = g.dim[0], cols = n0 + d;
            const double* M = g.tab + (int64_t)(g.fsys ? g.fsys[r.f] : 0) * g.tstride;
            for (int q = 0; q < d; ++q) {
                double acc = 0.0;
                for (int c = 0; c < cols; ++c) acc += M[q * cols + c] * (c < n0 ? v0[c] : v1[c - n0]);
                vio = fmax(vio, fabs(acc));
            }
            break;
        }
        case FG_KIND_SVM_SLACK: {            // operators.py:443-447
            const double v = zs(0)[0];
            obj = P[0] * (v > 0.0 ? v : 0.0);
            vio = -v > 0.0 ? -v : 0.0;
            break;
        }
        case FG_KIND_SVM_NORM: {             // operators.py:481-483
            const double* v = zs(0);
            double s = 0.0;
            for (int c = 0; c < g.dim[0]; ++c) s += v[c] * v[c];
            obj = 0.5 * P[0] * s;
            break;
        }
        case FG_KIND_SVM_MARGIN: {           // operators.py:527-532
            const double* w = zs(0);
            const int D = g.dim[0];
            double dot = 0.0;
            for (int c = 0; c < D; ++c) dot += w[c] * P[c];
            const double gap = (1.0 - zs(2)[0]) - P[D] * (dot + zs(1)[0]);
            vio = gap > 0.0 ? gap : 0.0;
            break;
        }
        case FG_KIND_EQUALITY: {             // operators.py:566-568
            const double* a1 = zs(0);
            const double* a2 = zs(1);
            for (int c = 0; c < g.dim[0]; ++c) vio = fmax(vio, fabs(a1[c] - a2[c]));
            break;
        }
        default:
            break;
    }
}

__global__ void __launch_bounds__(256) k_evaluate(GroupDev g, VarTab vt, const double* z,
                                                  double* part) {
    __shared__ double so[8], sv[8];
    double obj = 0.0, vio = 0.0;
    const int64_t total = g.count;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
         f += (int64_t)gridDim.x * blockDim.x) {
        // index-free addressing: translate the factor into its run
        FRef r{f, f, nullptr};
        if (g.runs) {
            int lo = 0, hi = g.nruns - 1;
            while (lo < hi) {                // last run with f0 <= f
                const int mid = (lo + hi + 1) >> 1;
                if (g.runs[mid].f0 <= f) lo = mid; else hi = mid - 1;
            }
            r.fl = f - g.runs[lo].f0;
            r.sr = g.sruns + (int64_t)lo * g.nslots;
        }
        double o, v;
        eval_factor(g, z, vt, r, o, v);
        obj += o;
        vio = fmax(vio, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        obj += __shfl_xor_sync(kFull, obj, o);
        vio = fmax(vio, __shfl_xor_sync(kFull, vio, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { so[w] = obj; sv[w] = vio; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < 8; ++i) { a += so[i]; b = fmax(b, sv[i]); }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}

}  // namespace fg
