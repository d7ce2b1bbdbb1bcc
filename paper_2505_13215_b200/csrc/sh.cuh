// sh.cuh -- real spherical-harmonics basis (degree <= 3) and its direction
// gradient in FP32 (sh.cpp:25-71), shared by K1 (colour + colour Jacobian)
// and K7b (SH backward).
#pragma once

namespace hgs {

// sh.cpp:25-47; T = float (K1 / K7b) or double (the exact refinement).
// The constants are written as double literals converted to T: for float
// they round to the same values as float literals.
template <typename T>
__device__ __forceinline__ void sh_basis_t(const T d[3], int deg, T out[16]) {
    const T x = d[0], y = d[1], z = d[2];
    out[0] = T(0.28209479177387814);
    if (deg < 1) return;
    out[1] = T(-0.4886025119029199) * y;
    out[2] = T(0.4886025119029199) * z;
    out[3] = T(-0.4886025119029199) * x;
    if (deg < 2) return;
    const T xx = x * x, yy = y * y, zz = z * z;
    out[4] = T(1.0925484305920792) * x * y;
    out[5] = T(-1.0925484305920792) * y * z;
    out[6] = T(0.31539156525252005) * (T(2) * zz - xx - yy);
    out[7] = T(-1.0925484305920792) * x * z;
    out[8] = T(0.5462742152960396) * (xx - yy);
    if (deg < 3) return;
    out[9] = T(-0.5900435899266435) * y * (T(3) * xx - yy);
    out[10] = T(2.890611442640554) * x * y * z;
    out[11] = T(-0.4570457994644658) * y * (T(4) * zz - xx - yy);
    out[12] = T(0.3731763325901154) * z * (T(2) * zz - T(3) * xx - T(3) * yy);
    out[13] = T(-0.4570457994644658) * x * (T(4) * zz - xx - yy);
    out[14] = T(1.445305721320277) * z * (xx - yy);
    out[15] = T(-0.5900435899266435) * x * (xx - T(3) * yy);
}
__device__ __forceinline__ void sh_basis_f(const float d[3], int deg, float out[16]) { sh_basis_t<float>(d, deg, out); }

// sum_k w_k * dY_k/d(dir) (sh.cpp:49-71) without materialising the 16x3 Jacobian
template <typename T>
__device__ __forceinline__ void sh_dir_grad_t(const T d[3], int deg, const T w[16], T g[3]) {
    const T x = d[0], y = d[1], z = d[2];
    g[0] = g[1] = g[2] = T(0);
    if (deg < 1) return;
    const T C1 = T(0.4886025119029199);
    g[1] -= C1 * w[1];
    g[2] += C1 * w[2];
    g[0] -= C1 * w[3];
    if (deg < 2) return;
    const T A = T(1.0925484305920792), B = T(0.31539156525252005), Cc = T(0.5462742152960396);
    g[0] += A * y * w[4];
    g[1] += A * x * w[4];
    g[1] -= A * z * w[5];
    g[2] -= A * y * w[5];
    g[0] += B * (T(-2) * x) * w[6];
    g[1] += B * (T(-2) * y) * w[6];
    g[2] += B * (T(4) * z) * w[6];
    g[0] -= A * z * w[7];
    g[2] -= A * x * w[7];
    g[0] += Cc * (T(2) * x) * w[8];
    g[1] += Cc * (T(-2) * y) * w[8];
    if (deg < 3) return;
    const T xx = x * x, yy = y * y, zz = z * z;
    const T D0 = T(-0.5900435899266435), D1 = T(2.890611442640554), D2 = T(-0.4570457994644658),
            D3 = T(0.3731763325901154), D5 = T(1.445305721320277);
    g[0] += D0 * (T(6) * x * y) * w[9];
    g[1] += D0 * (T(3) * xx - T(3) * yy) * w[9];
    g[0] += D1 * (y * z) * w[10];
    g[1] += D1 * (x * z) * w[10];
    g[2] += D1 * (x * y) * w[10];
    g[0] += D2 * (T(-2) * x * y) * w[11];
    g[1] += D2 * (T(4) * zz - xx - T(3) * yy) * w[11];
    g[2] += D2 * (T(8) * y * z) * w[11];
    g[0] += D3 * (T(-6) * x * z) * w[12];
    g[1] += D3 * (T(-6) * y * z) * w[12];
    g[2] += D3 * (T(6) * zz - T(3) * xx - T(3) * yy) * w[12];
    g[0] += D2 * (T(4) * zz - T(3) * xx - yy) * w[13];
    g[1] += D2 * (T(-2) * x * y) * w[13];
    g[2] += D2 * (T(8) * x * z) * w[13];
    g[0] += D5 * (T(2) * x * z) * w[14];
    g[1] += D5 * (T(-2) * y * z) * w[14];
    g[2] += D5 * (xx - yy) * w[14];
    g[0] += D0 * (T(3) * xx - T(3) * yy) * w[15];
    g[1] += D0 * (T(-6) * x * y) * w[15];
}
__device__ __forceinline__ void sh_dir_grad_f(const float d[3], int deg, const float w[16], float g[3]) {
    sh_dir_grad_t<float>(d, deg, w, g);
}

// dY_k / d(x, y, z) of one basis function (k a compile-time constant after
// unrolling), FP32 with explicit products for K1 (sh.cpp:49-71); entries
// outside sh_dir_nonzero are 0 and left unset.
__host__ __device__ constexpr bool sh_dir_nonzero(int k, int j) {
    // x / y / z dependence of Y_k
    return k == 0 ? false
         : k == 1 ? j == 1 : k == 2 ? j == 2 : k == 3 ? j == 0
         : k == 4 ? j != 2 : k == 5 ? j != 0 : k == 6 ? true : k == 7 ? j != 1 : k == 8 ? j != 2
         : k == 9 ? j != 2 : k == 15 ? j != 2 : true;
}
__device__ __forceinline__ void sh_dir_factor(int k, float x, float y, float z, float f[3]) {
    const float C1 = 0.4886025119029199f, A = 1.0925484305920792f, B = 0.31539156525252005f,
                Cc = 0.5462742152960396f, D0 = -0.5900435899266435f, D1 = 2.890611442640554f,
                D2 = -0.4570457994644658f, D3 = 0.3731763325901154f, D5 = 1.445305721320277f;
    switch (k) {
        case 1: f[1] = -C1; break;
        case 2: f[2] = C1; break;
        case 3: f[0] = -C1; break;
        case 4: f[0] = A * y; f[1] = A * x; break;
        case 5: f[1] = -A * z; f[2] = -A * y; break;
        case 6: f[0] = B * (-2.0f * x); f[1] = B * (-2.0f * y); f[2] = B * (4.0f * z); break;
        case 7: f[0] = -A * z; f[2] = -A * x; break;
        case 8: f[0] = Cc * (2.0f * x); f[1] = Cc * (-2.0f * y); break;
        case 9: f[0] = D0 * (6.0f * x * y); f[1] = D0 * (3.0f * x * x - 3.0f * y * y); break;
        case 10: f[0] = D1 * (y * z); f[1] = D1 * (x * z); f[2] = D1 * (x * y); break;
        case 11: f[0] = D2 * (-2.0f * x * y); f[1] = D2 * (4.0f * z * z - x * x - 3.0f * y * y); f[2] = D2 * (8.0f * y * z); break;
        case 12: f[0] = D3 * (-6.0f * x * z); f[1] = D3 * (-6.0f * y * z); f[2] = D3 * (6.0f * z * z - 3.0f * x * x - 3.0f * y * y); break;
        case 13: f[0] = D2 * (4.0f * z * z - 3.0f * x * x - y * y); f[1] = D2 * (-2.0f * x * y); f[2] = D2 * (8.0f * x * z); break;
        case 14: f[0] = D5 * (2.0f * x * z); f[1] = D5 * (-2.0f * y * z); f[2] = D5 * (x * x - y * y); break;
        case 15: f[0] = D0 * (3.0f * x * x - 3.0f * y * y); f[1] = D0 * (-6.0f * x * y); break;
        default: break;
    }
}

}  // namespace hgs
