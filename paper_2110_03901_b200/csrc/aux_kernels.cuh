// aux_kernels.cuh -- HBM-bound companions of the implicit kernel:
//   * explicit im2col (K3; the baseline whose overhead the paper quantifies),
//   * one decomposed tile's gather (TileDescriptor.gather_matrix),
//   * zero-padding copy used by the Python shim for 16-byte channel alignment.
// All are grid-stride copies with 16-byte vector accesses where the row
// length allows; row index m = (n*P + p)*Q + q (lowering.py:101-102).
#pragma once
#include <cstdint>

namespace imconv {

// Channel-first im2col / tap gather, 16-byte vector path.
// out[(m, col16)] where a row holds `taps` taps of c_vec 16-byte vectors.
// taps == 1 with fixed (r, s) is the tile gather.
__global__ void im2col_cf_vec16_kernel(const uint4 *__restrict__ x, uint4 *__restrict__ out, long long m_total,
                                       int h, int w, int c_vec, int p_, int q_, int r_lo, int s_lo, int taps,
                                       int wf, int sh, int sw, int ph, int pw, int dh, int dw) {
    const long long row_vec = static_cast<long long>(taps) * c_vec;
    const long long total = m_total * row_vec;
    const long long pq = static_cast<long long>(p_) * q_;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long m = idx / row_vec;
        const int rem = static_cast<int>(idx - m * row_vec);
        const int t = rem / c_vec;
        const int cv = rem - t * c_vec;
        const int n = static_cast<int>(m / pq);
        const int pqr = static_cast<int>(m - n * pq);
        const int op = pqr / q_;
        const int oq = pqr - op * q_;
        // r_lo >= 0: single fixed tap (tile gather); else tap t of a full im2col (t = 0 when hf*wf == 1)
        const int tap_r = r_lo >= 0 ? r_lo : t / wf;
        const int tap_s = r_lo >= 0 ? s_lo : t - (t / wf) * wf;
        const int hh = op * sh + tap_r * dh - ph;
        const int ww = oq * sw + tap_s * dw - pw;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (hh >= 0 && hh < h && ww >= 0 && ww < w)
            v = __ldg(&x[((static_cast<long long>(n) * h + hh) * w + ww) * c_vec + cv]);
        out[idx] = v;
    }
}

// Generic element-wise im2col (any element size, either column order);
// used for unaligned channel counts and the channel-last ordering.
template <typename T>
__global__ void im2col_generic_kernel(const T *__restrict__ x, T *__restrict__ out, long long m_total, int h, int w,
                                      int c, int p_, int q_, int hf, int wf, int sh, int sw, int ph, int pw, int dh,
                                      int dw, int channel_first, int r_fix, int s_fix) {
    // r_fix >= 0: single-tap gather (row length c), else full im2col (row length hf*wf*c)
    const long long kcols = r_fix >= 0 ? c : static_cast<long long>(hf) * wf * c;
    const long long total = m_total * kcols;
    const long long pq = static_cast<long long>(p_) * q_;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long m = idx / kcols;
        const int col = static_cast<int>(idx - m * kcols);
        int r, s, ch;
        if (r_fix >= 0) {
            r = r_fix;
            s = s_fix;
            ch = col;
        } else if (channel_first) {  // col = (r*wf + s)*c + ch
            ch = col % c;
            const int rs = col / c;
            r = rs / wf;
            s = rs % wf;
        } else {  // col = (ch*hf + r)*wf + s
            s = col % wf;
            const int cr = col / wf;
            r = cr % hf;
            ch = cr / hf;
        }
        const int n = static_cast<int>(m / pq);
        const int pqr = static_cast<int>(m - n * pq);
        const int op = pqr / q_;
        const int oq = pqr - op * q_;
        const int hh = op * sh + r * dh - ph;
        const int ww = oq * sw + s * dw - pw;
        T v = T(0);
        if (hh >= 0 && hh < h && ww >= 0 && ww < w) v = x[((static_cast<long long>(n) * h + hh) * w + ww) * c + ch];
        out[idx] = v;
    }
}

template <typename T>
__global__ void pad_copy_kernel(const T *__restrict__ src, T *__restrict__ dst, long long outer, int c, int d,
                                int c_pad, int d_pad) {
    const long long inner = static_cast<long long>(c_pad) * d_pad;
    const long long total = outer * inner;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long o = idx / inner;
        const int rem = static_cast<int>(idx - o * inner);
        const int ci = rem / d_pad;
        const int di = rem - ci * d_pad;
        T v = T(0);
        if (ci < c && di < d) v = src[(o * c + ci) * d + di];
        dst[idx] = v;
    }
}

// HWCN filter (R*S taps x C x K) -> channel-last reduction order (C x R*S x K):
// out[(c*RS + t)*K + k] = in[(t*C + c)*K + k]  (the B operand of the channel-last baseline)
template <typename T>
__global__ void permute_filter_cl_kernel(const T *__restrict__ in, T *__restrict__ out, int rs, int c, int k) {
    const long long total = static_cast<long long>(rs) * c * k;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = idx / k;
        const int kk = static_cast<int>(idx - row * k);
        const int ch = static_cast<int>(row / rs), t = static_cast<int>(row - static_cast<long long>(ch) * rs);
        out[idx] = in[(static_cast<long long>(t) * c + ch) * k + kk];
    }
}

}  // namespace imconv
