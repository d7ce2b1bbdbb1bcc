// train.cu -- training entry points of the C ABI (filled in next).
#include "train_api.cuh"
