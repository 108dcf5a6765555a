// Check-node kernels, degree bucket 24 (explicit instantiation unit).
#include "cnu_launch.cuh"

template int qcb::launch_cnu_dc<24>(const qc_plan*, const qcb::CnuArgs&, int, cudaStream_t);
