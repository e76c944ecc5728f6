// Probe (build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o dmma_check dmma_check.cu)
// Does mma.sync.m8n8k4 f64 reproduce a sequential fma chain over k bitwise?
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <random>
__global__ void k_dmma(const double* A, const double* B, const double* C, double* D, int nk) {
    // A: 8 x (4*nk) row-major, B: (4*nk) x 8 col-major (B[n*K + k]), C/D 8x8 row-major
    const int lane = threadIdx.x;
    const int K = 4 * nk;
    // accumulator fragment: row = lane/4, cols 2*(lane%4), +1
    const int r = lane >> 2, cpair = (lane & 3) * 2;
    double d0 = C[r * 8 + cpair], d1 = C[r * 8 + cpair + 1];
    for (int kb = 0; kb < nk; ++kb) {
        // A fragment (row-major 8x4): a = A[lane/4][lane%4]
        const double a = A[(lane >> 2) * K + kb * 4 + (lane & 3)];
        // B fragment (col-major 4x8): b = B[k = lane%4][n = lane/4]
        const double b = B[(lane >> 2) * K + kb * 4 + (lane & 3)];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    }
    D[r * 8 + cpair] = d0;
    D[r * 8 + cpair + 1] = d1;
}
__global__ void k_fma(const double* A, const double* B, const double* C, double* D, int nk) {
    const int t = threadIdx.x;
    if (t >= 64) return;
    const int r = t / 8, n = t % 8, K = 4 * nk;
    double acc = C[r * 8 + n];
    for (int k = 0; k < K; ++k) acc = __fma_rn(A[r * K + k], B[n * K + k], acc);
    D[r * 8 + n] = acc;
}
__global__ void k_fma_tree(const double* A, const double* B, const double* C, double* D, int nk) {
    // alternative: per k-block of 4, products summed then added?
    const int t = threadIdx.x;
    if (t >= 64) return;
    const int r = t / 8, n = t % 8, K = 4 * nk;
    double acc = C[r * 8 + n];
    for (int kb = 0; kb < nk; ++kb) {
        double s = 0;
        for (int k = 0; k < 4; ++k) s = __fma_rn(A[r * K + kb*4+k], B[n * K + kb*4+k], s);
        acc = acc + s;
    }
    D[r * 8 + n] = acc;
}
int main() {
    const int nk = 9, K = 36;
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd(0, 1);
    int mism = 0, mism2 = 0, trials = 2000;
    double *dA, *dB, *dC, *dD1, *dD2, *dD3;
    cudaMalloc(&dA, 8*K*8); cudaMalloc(&dB, 8*K*8); cudaMalloc(&dC, 64*8);
    cudaMalloc(&dD1, 64*8); cudaMalloc(&dD2, 64*8); cudaMalloc(&dD3, 64*8);
    double hA[8*36], hB[8*36], hC[64], h1[64], h2[64], h3[64];
    for (int t = 0; t < trials; ++t) {
        const int mode = t % 5;
        for (auto& v : hA) v = nd(g) * std::pow(10.0, (int)(nd(g)*3));
        for (auto& v : hB) v = nd(g);
        for (auto& v : hC) v = (t % 2) ? 0.0 : nd(g);
        if (mode == 1) {          // subnormal products / operands
            for (auto& v : hA) v *= 1e-300;
            for (auto& v : hB) v *= 1e-15;
        } else if (mode == 2) {   // a few infinities / NaNs / signed zeros
            hA[g() % 288] = INFINITY; hB[g() % 288] = -INFINITY; hA[g() % 288] = NAN;
            hB[g() % 288] = -0.0; hA[g() % 288] = 0.0; hC[g() % 64] = -0.0;
        } else if (mode == 3) {   // overflow
            for (auto& v : hA) v *= 1e300;
            for (auto& v : hB) v *= 1e10;
        } else if (mode == 4) {   // cancellation
            for (int i = 0; i < 288; i += 2) hA[i + 1] = -hA[i];
            for (int i = 0; i < 288; i += 2) hB[i + 1] = hB[i];
        }
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        cudaMemcpy(dC, hC, sizeof hC, cudaMemcpyHostToDevice);
        k_dmma<<<1, 32>>>(dA, dB, dC, dD1, nk);
        k_fma<<<1, 64>>>(dA, dB, dC, dD2, nk);
        k_fma_tree<<<1, 64>>>(dA, dB, dC, dD3, nk);
        cudaMemcpy(h1, dD1, sizeof h1, cudaMemcpyDeviceToHost);
        cudaMemcpy(h2, dD2, sizeof h2, cudaMemcpyDeviceToHost);
        cudaMemcpy(h3, dD3, sizeof h3, cudaMemcpyDeviceToHost);
        bool diff = false;
        for (int i = 0; i < 64; ++i) {
            const bool n1 = std::isnan(h1[i]), n2 = std::isnan(h2[i]);
            if (n1 != n2 || (!n1 && memcmp(&h1[i], &h2[i], 8))) diff = true;
        }
        if (diff) { ++mism; if (mism < 4) printf("mode %d differs\n", mode); }
        if (memcmp(h1, h3, sizeof h1)) ++mism2;
    }
    cudaError_t e = cudaGetLastError();
    printf("err=%s trials=%d dmma!=fma_chain: %d  dmma!=blocksum: %d\n", cudaGetErrorString(e), trials, mism, mism2);
    return 0;
}
