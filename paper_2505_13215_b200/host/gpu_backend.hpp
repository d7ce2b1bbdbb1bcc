// gpu_backend.hpp -- the reference's hot-path API (raster.hpp, backward.hpp,
// loss.hpp, train.hpp, scene.hpp of /root/reference/proj/include/hgs) with
// the B200 path behind it, through the C ABI of include/hgs_gpu.h.
//
// Compiled against the reference's own headers (and whatever Eigen the
// reference is built with).  By default the functions live in hgs::gpu, so
// a program can call the reference's CPU implementation and this one side by
// side (examples/backend_demo.cpp); with -DHGS_GPU_BACKEND_AS_HGS they are
// defined in namespace hgs itself -- a link-time drop-in for the reference's
// raster.cpp / backward.cpp / loss.cpp / train.cpp definitions of the same
// functions.
//
// Threading and state: one GPU context per host thread
// (device HGS_DEVICE, default 0).  forward_train leaves the tape on that
// context; the Tape object it fills is a handle (dimensions, time,
// background and a token), and backward() with a tape that is not the
// context's last one throws std::invalid_argument.  Status codes map to the
// reference's exception types (errors.hpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hgs/backward.hpp"
#include "hgs/loss.hpp"
#include "hgs/raster.hpp"
#include "hgs/scene.hpp"
#include "hgs/train.hpp"

#ifdef HGS_GPU_BACKEND_AS_HGS
#define HGS_GPU_NS hgs
#else
#define HGS_GPU_NS hgs::gpu
#endif

namespace HGS_GPU_NS {

// raster.hpp:79-80
RenderOutput rasterize(const HybridScene& scene, const Camera& cam, double t, const Vec3& background,
                       const RasterOpts& opts = {});
// raster.hpp:85-87
std::vector<uint32_t> density_map(const HybridScene& scene, const Camera& cam, double t, bool dynamics_only = false,
                                  double weight_cutoff = kDefaultWeightCutoff);
// backward.hpp:68-74
Image forward_train(const HybridScene& scene, const Camera& cam, double t, const Vec3& background,
                    const RasterOpts& opts, Tape& tape);
void backward(const HybridScene& scene, const Camera& cam, const Tape& tape, const Image& loss_grad,
              SceneGrads& grads);
// loss.hpp:12-13
double photometric_loss_with_grad(const Image& rendered, const Image& gt, double ssim_lambda, Image& grad);
// train.hpp:68-69
void optimizer_step(HybridScene& scene, const SceneGrads& grads, GradAccum& state, const LearningRates& lrs,
                    double mean_lr_scale = 1.0);
// scene.hpp:75
ConversionReport sweep_convert(HybridScene& scene, std::vector<std::size_t>* moved = nullptr);
// train.hpp:88-92: the device-resident training loop (train.cpp:382-494)
TrainResult train(const MultiViewDataset& dataset, const TrainConfig& cfg);
TrainResult train_scene(HybridScene scene, GradAccum state, const MultiViewDataset& dataset, const TrainConfig& cfg);

}  // namespace HGS_GPU_NS
