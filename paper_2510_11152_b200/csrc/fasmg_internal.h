// fasmg_internal.h -- host-side error plumbing shared by the .cu files.
#pragma once
#include <cuda_runtime.h>

#define FASMG_OK 0
#define FASMG_EINVAL 1001
#define FASMG_ECUDA 1002
#define FASMG_ENOMEM 1003
#define FASMG_ESTATE 1004

int fasmg_set_error(int code, const char* msg);
int fasmg_check_launch();        // cudaGetLastError -> status
int fasmg_check(cudaError_t e);  // status of a runtime call
