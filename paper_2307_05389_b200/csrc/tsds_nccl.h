// tsds_nccl.h -- run-time bound NCCL calls (tsds_nccl.cpp).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace tsds_nccl {

bool available(std::string* err);
std::string error_string(ncclResult_t r);
ncclResult_t get_unique_id(ncclUniqueId* id);
ncclResult_t comm_init_rank(ncclComm_t* c, int nranks, const ncclUniqueId& id, int rank);
ncclResult_t comm_destroy(ncclComm_t c);
ncclResult_t all_gather_bytes(const void* send, void* recv, size_t bytes, ncclComm_t c, cudaStream_t s);

}  // namespace tsds_nccl
