// comm.cpp -- the sharded layer's control plane and NCCL transport.
//
// Control plane (all-gather of small host messages, barrier) -- two implementations:
//   * NCCL 2.28 (venv) over NVLink 5 / NVSwitch (sv_create_sharded): bootstrap (N5),
//     ncclAllGather through a persistent device buffer, a one-word ncclAllReduce as the
//     stream-ordered barrier;
//   * host callbacks (sv_create_sharded_ex with an sv_control, e.g. torch.distributed over
//     gloo): stream synchronise + the caller's barrier.  This is what lets several processes
//     share ONE GPU (NCCL refuses two ranks on a device), so the real cross-process path --
//     CUDA IPC mapping, remote-store passes, flips -- runs in tests on a single B200.
// Data plane: peer-memory stores (sharded.cpp) or, NCCL only, pairwise ncclSend/ncclRecv of
// state chunks (N1/N2/N3).
#include <cstring>
#include <string>

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

// Persistent device buffer for the NCCL gathers (grown on demand, freed with the state).
static sv_status gather_buffer(sv_state_s* s, size_t bytes, std::string& err) {
    if (s->gather_bytes >= bytes) return SV_OK;
    if (s->d_gather) cudaFree(s->d_gather);
    s->d_gather = nullptr;
    s->gather_bytes = 0;
    if (cudaMalloc(&s->d_gather, bytes) != cudaSuccess) {
        cudaGetLastError();
        err = "cudaMalloc for the gather buffer failed (" + std::to_string(bytes) + " bytes)";
        return SV_ERR_RESOURCE;
    }
    s->gather_bytes = bytes;
    return SV_OK;
}

sv_status comm_allgather_bytes(sv_state_s* s, const void* local, size_t bytes, std::vector<unsigned char>& all,
                               std::string& err) {
    all.assign(bytes * s->world, 0);
    if (s->host_ctl) {
        // host control plane (sv_create_sharded_ex with an sv_control): the caller's all-gather
        if (s->ctl.allgather(s->ctl.user, local, bytes, all.data()) != 0) {
            err = "sv_control.allgather failed";
            return SV_ERR_NCCL;
        }
        return SV_OK;
    }
    sv_status st = gather_buffer(s, bytes * (s->world + 1), err);
    if (st != SV_OK) return st;
    unsigned char* d = (unsigned char*)s->d_gather;
    cudaError_t e = cudaMemcpyAsync(d, local, bytes, cudaMemcpyHostToDevice, s->stream);
    if (e != cudaSuccess) {
        err = std::string("allgather upload: ") + cudaGetErrorString(e);
        return SV_ERR_CUDA;
    }
    const ncclResult_t r = ncclAllGather(d, d + bytes, bytes, ncclUint8, (ncclComm_t)s->comm, s->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather", err);
    e = cudaMemcpyAsync(all.data(), d + bytes, bytes * s->world, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) {
        err = std::string("allgather: ") + cudaGetErrorString(e);
        return SV_ERR_CUDA;
    }
    return SV_OK;
}

sv_status comm_allgather_doubles(sv_state_s* s, const double* local, size_t count, std::vector<double>& all,
                                 std::string& err) {
    std::vector<unsigned char> raw;
    const sv_status st = comm_allgather_bytes(s, local, count * sizeof(double), raw, err);
    if (st != SV_OK) return st;
    all.resize(count * s->world);
    std::memcpy(all.data(), raw.data(), raw.size());
    return SV_OK;
}

sv_status comm_barrier(sv_state_s* s, std::string& err) {
    if (s->host_ctl) {
        // host control plane: every rank's launched work (its stores into peer memory
        // included) completes before the host barrier lets anyone continue
        const cudaError_t e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess) {
            err = std::string("barrier: ") + cudaGetErrorString(e);
            return SV_ERR_CUDA;
        }
        if (s->ctl.barrier(s->ctl.user) != 0) {
            err = "sv_control.barrier failed";
            return SV_ERR_NCCL;
        }
        return SV_OK;
    }
    const ncclResult_t r = ncclAllReduce(s->xflag, s->xflag, 1, ncclInt32, ncclSum, (ncclComm_t)s->comm, s->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce (barrier)", err);
    return SV_OK;
}

}  // namespace svb
