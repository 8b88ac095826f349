// comm.cpp -- NCCL 2.28 (venv) over NVLink 5 / NVSwitch: bootstrap (N5), pairwise
// exchange of state chunks (N1/N2/N3), rank-ordered gather of fp64 partials (N4).
#include <cstring>

#include <nccl.h>

#include "comm.hpp"

namespace svb {

static sv_status nccl_fail(ncclResult_t r, const char* where, std::string& err) {
    err = std::string(where) + ": " + ncclGetErrorString(r);
    return SV_ERR_NCCL;
}

sv_status comm_unique_id(void* out, std::string& err) {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId", err);
    static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
    std::memcpy(out, &id, sizeof id);
    return SV_OK;
}

sv_status comm_init(void** comm, const void* uid, int world, int rank, std::string& err) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclComm_t c;
    const ncclResult_t r = ncclCommInitRank(&c, world, id, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank", err);
    *comm = c;
    return SV_OK;
}

void comm_destroy(void* comm) {
    if (comm) ncclCommDestroy((ncclComm_t)comm);
}

sv_status comm_sendrecv(sv_state_s* s, int peer, const void* send, void* recv, size_t bytes, std::string& err) {
    ncclComm_t c = (ncclComm_t)s->comm;
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess) r = ncclSend(send, bytes, ncclUint8, peer, c, s->stream);
    if (r == ncclSuccess) r = ncclRecv(recv, bytes, ncclUint8, peer, c, s->stream);
    const ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv", err);
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd", err);
    return SV_OK;
}

sv_status comm_allgather_doubles(sv_state_s* s, const double* local, size_t count, std::vector<double>& all,
                                 std::string& err) {
    double* d = nullptr;
    const size_t bytes = count * sizeof(double);
    if (cudaMalloc(&d, bytes * (s->world + 1)) != cudaSuccess) {
        err = "cudaMalloc for the gather buffer failed";
        return SV_ERR_CUDA;
    }
    cudaMemcpyAsync(d, local, bytes, cudaMemcpyHostToDevice, s->stream);
    const ncclResult_t r = ncclAllGather(d, d + count, count, ncclDouble, (ncclComm_t)s->comm, s->stream);
    all.assign(count * s->world, 0.0);
    cudaMemcpyAsync(all.data(), d + count, bytes * s->world, cudaMemcpyDeviceToHost, s->stream);
    const cudaError_t e = cudaStreamSynchronize(s->stream);
    cudaFree(d);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather", err);
    if (e != cudaSuccess) {
        err = std::string("allgather: ") + cudaGetErrorString(e);
        return SV_ERR_CUDA;
    }
    return SV_OK;
}

sv_status comm_allgather_bytes(sv_state_s* s, const void* local, size_t bytes, std::vector<unsigned char>& all,
                               std::string& err) {
    unsigned char* d = nullptr;
    if (cudaMalloc(&d, bytes * (s->world + 1)) != cudaSuccess) {
        cudaGetLastError();
        err = "cudaMalloc for the gather buffer failed";
        return SV_ERR_CUDA;
    }
    cudaMemcpyAsync(d, local, bytes, cudaMemcpyHostToDevice, s->stream);
    const ncclResult_t r = ncclAllGather(d, d + bytes, bytes, ncclUint8, (ncclComm_t)s->comm, s->stream);
    all.assign(bytes * s->world, 0);
    cudaMemcpyAsync(all.data(), d + bytes, bytes * s->world, cudaMemcpyDeviceToHost, s->stream);
    const cudaError_t e = cudaStreamSynchronize(s->stream);
    cudaFree(d);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather", err);
    if (e != cudaSuccess) {
        err = std::string("allgather: ") + cudaGetErrorString(e);
        return SV_ERR_CUDA;
    }
    return SV_OK;
}

sv_status comm_barrier(sv_state_s* s, std::string& err) {
    const ncclResult_t r = ncclAllReduce(s->xflag, s->xflag, 1, ncclInt32, ncclSum, (ncclComm_t)s->comm, s->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce (barrier)", err);
    return SV_OK;
}

}  // namespace svb
