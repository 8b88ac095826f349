// comm.hpp -- multi-GPU layer: NCCL plumbing (comm.cpp) and the sharded run loop with its
// global<->local qubit swaps (sharded.cpp).  SURVEY 8(e); PAPER.md:123 (multi-GPU is the
// paper's stated future work), PAPER.md:55 (communication is the large-n bottleneck).
#pragma once
#include <string>
#include <vector>

#include "state.hpp"

namespace svb {

sv_status comm_unique_id(void* out_128B, std::string& err);
sv_status comm_init(void** comm, const void* uid_128B, int world, int rank, std::string& err);
void comm_destroy(void* comm);
// grouped ncclSend(send -> peer) + ncclRecv(recv <- peer) of `bytes` on the state's stream
sv_status comm_sendrecv(sv_state_s* s, int peer, const void* send, void* recv, size_t bytes, std::string& err);
// every rank's `count` doubles, gathered in rank order (host in/out)
sv_status comm_allgather_doubles(sv_state_s* s, const double* local, size_t count, std::vector<double>& all,
                                 std::string& err);

// every rank's `bytes` host bytes, gathered in rank order (host in/out)
sv_status comm_allgather_bytes(sv_state_s* s, const void* local, size_t bytes, std::vector<unsigned char>& all,
                               std::string& err);
// stream-ordered barrier: a one-word all-reduce on the state's stream (every rank's earlier
// kernels, including their stores into peer memory, complete before anyone's later ones start)
sv_status comm_barrier(sv_state_s* s, std::string& err);

}  // namespace svb

sv_status sharded_apply(sv_state_s* s, sv_plan_s* p, sv_run_stats* stats);
sv_status sharded_canonicalize(sv_state_s* s);
