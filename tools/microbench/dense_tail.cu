// Microbenchmark (profiling aid): the inverse dense-tail passes of one rank
// (T = 32, nr = 6 rows) on one CTA of 256 threads, timed with clock64 inside
// the kernel, several variants.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }
__device__ __forceinline__ int tail_col_level(int col) { return 1 << ilog2(col + 2); }

template <typename T, int NRM>
__device__ void s1b(const T* Et, const T* zt, int pz, int Tt, int r0, int nr, T* U) {
    const int ncol = 2 * Tt - 2, ep = Tt + 1;
    int ri[NRM];
#pragma unroll
    for (int i = 0; i < NRM; ++i) ri[i] = (r0 + i) & (Tt - 1);
    for (int base = 0; base < 4 * ncol; base += blockDim.x) {
        const int e = base + threadIdx.x;
        const int col = e >> 2, g = e & 3;
        T acc[NRM];
#pragma unroll
        for (int i = 0; i < NRM; ++i) acc[i] = T(0);
        if (col < ncol) {
            const int s = tail_col_level(col), h = s >> 1, b = col - (s - 2);
            const int a0 = (b < h && s > 2) ? h : 0;
            for (int a = a0 + g; a < s; a += 4) {
                const T zv = zt[a * pz + b];
                const T* er = Et + (s - 2 + a) * ep;
#pragma unroll
                for (int i = 0; i < NRM; ++i)
                    if (i < nr) acc[i] += er[ri[i]] * zv;
            }
        }
#pragma unroll
        for (int i = 0; i < NRM; ++i) {
            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 1);
            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 2);
        }
        if (col < ncol && g == 0) {
#pragma unroll
            for (int i = 0; i < NRM; ++i)
                if (i < nr) U[i * ncol + col] = acc[i];
        }
    }
}
template <typename T, int NRM>
__device__ void s2b(const T* Et, int Tt, int nr, const T* U, T* red, T* out, int pout) {
    const int ncol = 2 * Tt - 2, ep = Tt + 1, lt = ilog2(Tt);
    const int G = blockDim.x >> lt, c = threadIdx.x & (Tt - 1), g = threadIdx.x >> lt;
    T acc[NRM];
#pragma unroll
    for (int i = 0; i < NRM; ++i) acc[i] = T(0);
    for (int col = g; col < ncol; col += G) {
        const T ev = Et[col * ep + c];
#pragma unroll
        for (int i = 0; i < NRM; ++i)
            if (i < nr) acc[i] += U[i * ncol + col] * ev;
    }
#pragma unroll
    for (int i = 0; i < NRM; ++i)
        if (i < nr) red[(g * nr + i) * Tt + c] = acc[i];
    __syncthreads();
    for (int e = threadIdx.x; e < nr * Tt; e += blockDim.x) {
        const int i = e >> lt, cc = e & (Tt - 1);
        T v = red[i * Tt + cc];
        for (int k = 1; k < G; ++k) v += red[(k * nr + i) * Tt + cc];
        out[i * pout + cc] = v;
    }
}

template <typename T, int NR, int PART>
__device__ void s2x(const T* Et, int Tt, const T* U, T* red, T* out, int pout) {
    const int ncol = 2 * Tt - 2, ep = Tt + 1, lt = ilog2(Tt);
    const int G = blockDim.x >> lt, c = threadIdx.x & (Tt - 1), g = threadIdx.x >> lt;
    T acc[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[i] = T(0);
    if (PART & 1) {
        for (int col = g; col < ncol; col += G) {
            const T ev = Et[col * ep + c];
#pragma unroll
            for (int i = 0; i < NR; ++i) acc[i] += U[i * ncol + col] * ev;
        }
    }
#pragma unroll
    for (int i = 0; i < NR; ++i) red[(g * NR + i) * Tt + c] = acc[i];
    __syncthreads();
    if (PART & 2) {
        for (int e = threadIdx.x; e < NR * Tt; e += blockDim.x) {
            const int i = e >> lt, cc = e & (Tt - 1);
            T v = red[i * Tt + cc];
            for (int k = 1; k < G; ++k) v += red[(k * NR + i) * Tt + cc];
            out[i * pout + cc] = v;
        }
    }
}

template <typename T, int NR>
__device__ void s2y(const T* Et, int Tt, const T* U, T* red, T* out, int pout) {
    const int ncol = 2 * Tt - 2, ep = Tt + 1, lt = ilog2(Tt);
    const int G = blockDim.x >> lt, c = threadIdx.x & (Tt - 1), g = threadIdx.x >> lt;
    T acc[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[i] = T(0);
    int col = g;
    for (; col + G < ncol; col += 2 * G) {
        T u0[NR], u1[NR];
        const T e0 = Et[col * ep + c], e1 = Et[(col + G) * ep + c];
#pragma unroll
        for (int i = 0; i < NR; ++i) { u0[i] = U[i * ncol + col]; u1[i] = U[i * ncol + col + G]; }
#pragma unroll
        for (int i = 0; i < NR; ++i) acc[i] += u0[i] * e0;
#pragma unroll
        for (int i = 0; i < NR; ++i) acc[i] += u1[i] * e1;
    }
    if (col < ncol) {
        T u0[NR];
        const T e0 = Et[col * ep + c];
#pragma unroll
        for (int i = 0; i < NR; ++i) u0[i] = U[i * ncol + col];
#pragma unroll
        for (int i = 0; i < NR; ++i) acc[i] += u0[i] * e0;
    }
#pragma unroll
    for (int i = 0; i < NR; ++i) red[(g * NR + i) * Tt + c] = acc[i];
    __syncthreads();
    for (int e = threadIdx.x; e < NR * Tt; e += blockDim.x) {
        const int i = e >> lt, cc = e & (Tt - 1);
        T v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = k < G ? red[(k * NR + i) * Tt + cc] : T(0);
        T sacc = v[0];
#pragma unroll
        for (int k = 1; k < 8; ++k) sacc += v[k];
        out[i * pout + cc] = sacc;
    }
}
template <typename T, int NRM>
__device__ void s1y(const T* Et, const T* zt, int pz, int Tt, int r0, int nr, T* U) {
    const int ncol = 2 * Tt - 2, ep = Tt + 1;
    int ri[NRM];
#pragma unroll
    for (int i = 0; i < NRM; ++i) ri[i] = (r0 + i) & (Tt - 1);
    for (int base = 0; base < 4 * ncol; base += blockDim.x) {
        const int e = base + threadIdx.x;
        const int col = e >> 2, g = e & 3;
        T acc[NRM];
#pragma unroll
        for (int i = 0; i < NRM; ++i) acc[i] = T(0);
        if (col < ncol) {
            const int s = tail_col_level(col), h = s >> 1, b = col - (s - 2);
            const int a0 = (b < h && s > 2) ? h : 0;
            for (int a = a0 + g; a < s; a += 4) {
                const T zv = zt[a * pz + b];
                const T* er = Et + (s - 2 + a) * ep;
                T ev[NRM];
#pragma unroll
                for (int i = 0; i < NRM; ++i) ev[i] = er[ri[i]];
#pragma unroll
                for (int i = 0; i < NRM; ++i) acc[i] += ev[i] * zv;
            }
        }
#pragma unroll
        for (int i = 0; i < NRM; ++i) {
            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 1);
            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 2);
        }
        if (col < ncol && g == 0) {
#pragma unroll
            for (int i = 0; i < NRM; ++i)
                if (i < nr) U[i * ncol + col] = acc[i];
        }
    }
}

// stage 2, contiguous column chunks per warp, 128-bit broadcast loads of U
template <typename T, int NR>
__device__ void s2z(const T* Et, int Tt, const T* U, T* red, T* out, int pout) {
    const int ncol = 2 * Tt - 2, ep = Tt + 1, lt = ilog2(Tt);
    const int G = blockDim.x >> lt, c = threadIdx.x & (Tt - 1), g = threadIdx.x >> lt;
    const int cw = ((ncol + G - 1) / G + 1) & ~1;  // columns per group (even)
    const int c0 = g * cw, c1 = min(c0 + cw, ncol);
    T acc[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[i] = T(0);
    for (int col = c0; col < c1; col += 2) {  // ncol and cw even
        const T e0 = Et[col * ep + c], e1 = Et[(col + 1) * ep + c];
        double2 u[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) u[i] = *reinterpret_cast<const double2*>(U + i * ncol + col);
#pragma unroll
        for (int i = 0; i < NR; ++i) acc[i] += u[i].x * e0 + u[i].y * e1;
    }
#pragma unroll
    for (int i = 0; i < NR; ++i) red[(g * NR + i) * Tt + c] = acc[i];
    __syncthreads();
    for (int e = threadIdx.x; e < NR * Tt; e += blockDim.x) {
        const int i = e >> lt, cc = e & (Tt - 1);
        T v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = k < G ? red[(k * NR + i) * Tt + cc] : T(0);
        out[i * pout + cc] = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    }
}
// stage 1 by level: warp w < 4 -> level 32, a in [8w, 8w+8); warp 4 -> level 16 (lanes: b + 16 * chunk,
// a in chunk*8..+8); warp 5 -> levels 2..8 (lane = col); partials P[k][i][col] (k < 4), summed in stage 2
template <typename T, int NR>
__device__ void s1z(const T* Et, const T* zt, int pz, int Tt, int r0, T* P) {
    const int ncol = 2 * Tt - 2, ep = Tt + 1;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int ri[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) ri[i] = (r0 + i) & (Tt - 1);
    T acc[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[i] = T(0);
    int s, b, alo, ahi, k, col;
    if (w < 4) { s = 32; b = lane; k = w; alo = 8 * w; ahi = alo + 8; if (b < 16 && alo < 16) alo = ahi; }
    else if (w == 4) { s = 16; b = lane & 15; k = lane >> 4; alo = 8 * k; ahi = alo + 8; if (b < 8 && alo < 8) alo = ahi; }
    else if (w == 5 && lane < 14) {
        col = lane; s = tail_col_level(col); b = col - (s - 2); k = 0;
        const int h = s >> 1; alo = (b < h && s > 2) ? h : 0; ahi = s;
    } else { s = 0; b = 0; k = 0; alo = ahi = 0; }
    for (int a = alo; a < ahi; ++a) {
        const T zv = zt[a * pz + b];
        const T* er = Et + (s - 2 + a) * ep;
        T ev[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) ev[i] = er[ri[i]];
#pragma unroll
        for (int i = 0; i < NR; ++i) acc[i] += ev[i] * zv;
    }
    if (w < 6 && s > 0) {
        col = s - 2 + b;
#pragma unroll
        for (int i = 0; i < NR; ++i) P[(k * NR + i) * ncol + col] = acc[i];
    }
}
template <int V>
__global__ void k(const double* g_et, const double* g_z, double* g_out, long long* cyc, int reps) {
    __shared__ double Et[62 * 33 + 4], Z[32 * 32], U[6 * 62], red[256 * 6 + 4 * 6 * 62], out[6 * 33];
    for (int e = threadIdx.x; e < 62 * 33; e += blockDim.x) Et[e] = g_et[e];
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) Z[e] = g_z[e];
    for (int e = threadIdx.x; e < 6 * 62; e += blockDim.x) U[e] = 0;
    __syncthreads();
    long long t0 = 0;
    for (int r = 0; r <= reps; ++r) {
        if (r == 1) t0 = clock64();
        if (V == 0) s1b<double, 6>(Et, Z, 32, 32, 4 * blockIdx.x - 2 + r, 6, U);
        if (V == 1) s2b<double, 6>(Et, 32, 6, U, red, out, 33);
        if (V == 3) s2x<double, 6, 3>(Et, 32, U, red, out, 33);
        if (V == 4) s2x<double, 6, 1>(Et, 32, U, red, out, 33);
        if (V == 5) s2x<double, 6, 2>(Et, 32, U, red, out, 33);
        if (V == 6) s2x<double, 6, 0>(Et, 32, U, red, out, 33);
        if (V == 7) s2y<double, 6>(Et, 32, U, red, out, 33);
        if (V == 8) s1y<double, 6>(Et, Z, 32, 32, 4 * blockIdx.x - 2 + r, 6, U);
        if (V == 9) s2z<double, 6>(Et, 32, U, red, out, 33);
        if (V == 10) s1z<double, 6>(Et, Z, 32, 32, 4 * blockIdx.x - 2 + r, red);
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
    if (threadIdx.x < 6 * 33) g_out[blockIdx.x * 256 + threadIdx.x] = out[threadIdx.x] + U[threadIdx.x % 372];
}
int main() {
    double *et, *z, *o; long long* c;
    cudaMalloc(&et, 62 * 33 * 8); cudaMalloc(&z, 32 * 32 * 8); cudaMalloc(&o, 148 * 256 * 8); cudaMalloc(&c, 148 * 8);
    cudaMemset(et, 0, 62 * 33 * 8); cudaMemset(z, 0, 32 * 32 * 8);
    long long h[148];
    for (int rep = 0; rep < 2; ++rep) {
        for (int v = 0; v < 11; ++v) {
            if (v == 9) k<9><<<72, 256>>>(et, z, o, c, 20);
            if (v == 10) k<10><<<72, 256>>>(et, z, o, c, 20);
            if (v == 7) k<7><<<72, 256>>>(et, z, o, c, 20);
            if (v == 8) k<8><<<72, 256>>>(et, z, o, c, 20);
            if (v == 0) k<0><<<72, 256>>>(et, z, o, c, 20);
            if (v == 1) k<1><<<72, 256>>>(et, z, o, c, 20);
            if (v == 2) k<2><<<72, 256>>>(et, z, o, c, 20);
            if (v == 3) k<3><<<72, 256>>>(et, z, o, c, 20);
            if (v == 4) k<4><<<72, 256>>>(et, z, o, c, 20);
            if (v == 5) k<5><<<72, 256>>>(et, z, o, c, 20);
            if (v == 6) k<6><<<72, 256>>>(et, z, o, c, 20);
            cudaMemcpy(h, c, 72 * 8, cudaMemcpyDeviceToHost);
            long long mx = 0, s = 0;
            for (int i = 0; i < 72; ++i) { mx = h[i] > mx ? h[i] : mx; s += h[i]; }
            if (rep) printf("variant %d: mean %lld max %lld cycles per pass (incl. one barrier)\n", v, s / 72, mx);
        }
    }
    return 0;
}
