// Internal declarations shared by the libsmpm translation units.
#pragma once
#include <cuda_runtime.h>

// Records the message returned by smpm_last_error() (thread-local).
void smpm_internal_set_error(const char* msg);
