// flr_common.cuh -- shared compile-time layout of the FLR workspace (sm_100a path).
//
// Component layout of one block's moments (X^T X is split
// into n, u_X and S; X^T Y's top row holds n mu_Y):
//   [0]                 n      = number of pixels of the block (exact integer)
//   [1 .. Q]            u_j    = sum x_j
//   [C_S .. +NS)        S_ij   = sum x_i x_j, i <= j, row-major upper triangle
//   [C_Y .. +3)         Y_c    = sum y_c
//   [C_XY .. +3Q)       XY_jc  = sum x_j y_c  (index j*3 + c)
//   [C_SH .. +Q)        c_j    = per-block shift (raw fp32 moments only)
// The raw (K1) moments are taken about the shift c (x - c, design rule H1 of
// DESIGN.md); the fp64 moments (after un-shifting) use indices [0, KM).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace flr {

constexpr int kMaxQ = 15;
constexpr int kMaxR = 32;  // blur half-width cap in blocks

template <int Q>
struct Dims {
    static constexpr int P = Q + 1;
    static constexpr int NS = Q * (Q + 1) / 2;
    static constexpr int C_N = 0;
    static constexpr int C_U = 1;
    static constexpr int C_S = 1 + Q;
    static constexpr int C_Y = C_S + NS;
    static constexpr int C_XY = C_Y + 3;
    static constexpr int C_SH = C_XY + 3 * Q;
    static constexpr int KM = C_SH;       // fp64 moment components
    static constexpr int KRAW = C_SH + Q; // raw fp32 components incl. shift
    static constexpr int MSTRIDE = ((3 * P + 3) / 4) * 4;  // padded model floats (16 B multiple)
    __host__ __device__ static constexpr int s_idx(int i, int j)  // i <= j
    {
        return C_S + i * Q - (i * (i - 1)) / 2 + (j - i);
    }
};

inline int km_of(int Q) { return 1 + Q + Q * (Q + 1) / 2 + 3 + 3 * Q; }
inline int kraw_of(int Q) { return km_of(Q) + Q; }
inline int mstride_of(int Q) { return ((3 * (Q + 1) + 3) / 4) * 4; }

// compile-time loop: f(integral_constant<int, 0>) ... f(integral_constant<int, N-1>), so every
// array index below is a constant and the factor stays in registers
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f)
{
    if constexpr (N > 0) {
        static_for<N - 1>(f);
        f(std::integral_constant<int, N - 1>{});
    }
}

struct Taps {
    double g[2 * kMaxR + 1];  // g[R + i] = exp(-i^2 / (2 s^2))
    int R;
};

}  // namespace flr
