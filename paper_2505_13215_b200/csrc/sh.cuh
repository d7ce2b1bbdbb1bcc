// sh.cuh -- real spherical-harmonics basis (degree <= 3) and its direction
// gradient in FP32 (sh.cpp:25-71), shared by K1 (colour + colour Jacobian)
// and K7b (SH backward).
#pragma once

namespace hgs {

// sh.cpp:25-47 in FP32
__device__ __forceinline__ void sh_basis_f(const float d[3], int deg, float out[16]) {
    const float x = d[0], y = d[1], z = d[2];
    out[0] = 0.28209479177387814f;
    if (deg < 1) return;
    out[1] = -0.4886025119029199f * y;
    out[2] = 0.4886025119029199f * z;
    out[3] = -0.4886025119029199f * x;
    if (deg < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    out[4] = 1.0925484305920792f * x * y;
    out[5] = -1.0925484305920792f * y * z;
    out[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    out[7] = -1.0925484305920792f * x * z;
    out[8] = 0.5462742152960396f * (xx - yy);
    if (deg < 3) return;
    out[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    out[10] = 2.890611442640554f * x * y * z;
    out[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    out[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    out[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    out[14] = 1.445305721320277f * z * (xx - yy);
    out[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

// sum_k w_k * dY_k/d(dir) (sh.cpp:49-71) without materialising the 16x3 Jacobian
__device__ __forceinline__ void sh_dir_grad_f(const float d[3], int deg, const float w[16], float g[3]) {
    const float x = d[0], y = d[1], z = d[2];
    g[0] = g[1] = g[2] = 0.0f;
    if (deg < 1) return;
    const float C1 = 0.4886025119029199f;
    g[1] -= C1 * w[1];
    g[2] += C1 * w[2];
    g[0] -= C1 * w[3];
    if (deg < 2) return;
    const float A = 1.0925484305920792f, B = 0.31539156525252005f, Cc = 0.5462742152960396f;
    g[0] += A * y * w[4];
    g[1] += A * x * w[4];
    g[1] -= A * z * w[5];
    g[2] -= A * y * w[5];
    g[0] += B * (-2.0f * x) * w[6];
    g[1] += B * (-2.0f * y) * w[6];
    g[2] += B * (4.0f * z) * w[6];
    g[0] -= A * z * w[7];
    g[2] -= A * x * w[7];
    g[0] += Cc * (2.0f * x) * w[8];
    g[1] += Cc * (-2.0f * y) * w[8];
    if (deg < 3) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    const float D0 = -0.5900435899266435f, D1 = 2.890611442640554f, D2 = -0.4570457994644658f,
                D3 = 0.3731763325901154f, D5 = 1.445305721320277f;
    g[0] += D0 * (6.0f * x * y) * w[9];
    g[1] += D0 * (3.0f * xx - 3.0f * yy) * w[9];
    g[0] += D1 * (y * z) * w[10];
    g[1] += D1 * (x * z) * w[10];
    g[2] += D1 * (x * y) * w[10];
    g[0] += D2 * (-2.0f * x * y) * w[11];
    g[1] += D2 * (4.0f * zz - xx - 3.0f * yy) * w[11];
    g[2] += D2 * (8.0f * y * z) * w[11];
    g[0] += D3 * (-6.0f * x * z) * w[12];
    g[1] += D3 * (-6.0f * y * z) * w[12];
    g[2] += D3 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * w[12];
    g[0] += D2 * (4.0f * zz - 3.0f * xx - yy) * w[13];
    g[1] += D2 * (-2.0f * x * y) * w[13];
    g[2] += D2 * (8.0f * x * z) * w[13];
    g[0] += D5 * (2.0f * x * z) * w[14];
    g[1] += D5 * (-2.0f * y * z) * w[14];
    g[2] += D5 * (xx - yy) * w[14];
    g[0] += D0 * (3.0f * xx - 3.0f * yy) * w[15];
    g[1] += D0 * (-6.0f * x * y) * w[15];
}

}  // namespace hgs
