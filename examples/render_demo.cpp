// render_demo.cpp -- a plain C++ consumer of the C ABI (no torch, no CUDA
// headers): uploads a one-Gaussian scene, renders it, prints the centre pixel.
//   g++ -std=c++17 -I include examples/render_demo.cpp
//       -L paper_2505_13215_b200 -lhgs_gpu -Wl,-rpath,$PWD/paper_2505_13215_b200 -o render_demo
#include <cmath>
#include <cstdio>
#include <vector>

#include "hgs_gpu.h"

int main() {
    hgs_ctx* ctx = nullptr;
    if (hgs_ctx_create(0, &ctx) != HGS_OK) {
        std::fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    // one static Gaussian at the origin, SH degree 0 (scene.hpp:27-36)
    double mean[3] = {0, 0, 0}, quat[4] = {1, 0, 0, 0}, ls[3] = {std::log(0.3), std::log(0.3), std::log(0.3)};
    double op = std::log(0.7 / 0.3), sh[3] = {(0.9 - 0.5) / 0.28209479177387814, (0.1 - 0.5) / 0.28209479177387814,
                                              (0.3 - 0.5) / 0.28209479177387814};
    hgs_host_scene s{0, 1, 0, 0.5, 1.0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                     mean, quat, ls, &op, sh};
    // camera at (0,0,-3) looking at the origin, up (0,-1,0) (camera.cpp:6-22)
    hgs_camera cam{40, 40, 16.5, 16.5, {1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 0, 3}, 33, 33, 0.01, 100.0};
    const double bg[3] = {0, 0, 1};
    hgs_raster_opts opts{0.05, 1, 0, 0};
    std::vector<double> rgb(33 * 33 * 3);
    hgs_render_stats st{};
    if (hgs_rasterize(ctx, &s, HGS_F64, &cam, 0.0, bg, &opts, rgb.data(), nullptr, nullptr, &st) != HGS_OK) {
        std::fprintf(stderr, "rasterize failed: %s\n", hgs_last_error(ctx));
        return 1;
    }
    const size_t c = (16 * 33 + 16) * 3;
    std::printf("projected=%lld centre=(%.6f, %.6f, %.6f)\n", (long long)st.projected, rgb[c], rgb[c + 1], rgb[c + 2]);
    hgs_ctx_destroy(ctx);
    return 0;
}
