// dm.cu -- device data manager (placeholder; filled in below)
#include "common.cuh"
