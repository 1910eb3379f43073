// comm.h -- internal NCCL hop transport used by runtime.cu (see comm.cu).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include "coe_cuda.h"

bool coe_comm_send_bf16(coe_comm *c, const void *buf, size_t count, int peer, cudaStream_t stream);
bool coe_comm_recv_bf16(coe_comm *c, void *buf, size_t count, int peer, cudaStream_t stream);
int coe_comm_rank(const coe_comm *c);
bool coe_comm_group(coe_comm *c, bool start);  // ncclGroupStart / ncclGroupEnd (no-op in-process)

// fused peer hops inside one process (see comm.cu)
bool coe_hub_publish(coe_local_hub *hub, int64_t key, cudaStream_t stream);
bool coe_hub_wait(coe_local_hub *hub, int64_t key, cudaStream_t stream);
