// Slab-rank collectives of one context (slabcomm.cu): the Arnoldi dot / norm all-reduces and
// the x-halo exchange, issued from C on the context's streams.
//
// Two transports behind one interface:
//  * NCCL (one process per GPU over NVLink / NVSwitch): libnccl is bound at run time (the one
//    torch already loaded, else the system's), two communicators per context — one for the
//    stream-ordered all-reduces on the compute stream, one for the halo exchange on its own
//    stream so it overlaps the interior stencil rows;
//  * host callbacks (tests: several ranks sharing one GPU through a CPU transport): the
//    collective synchronises the stream, stages through pinned memory and calls back.
#pragma once
#include "emhd_common.cuh"

namespace emhd {

typedef int (*HostAllreduceFn)(void* user, double* buf, int n, int op);             // op 0 sum, 2 max
typedef int (*HostExchangeFn)(void* user, const double* send, double* recv, long long n_side);

struct SlabComm;

// NCCL: unique ids come from rank 0 (emhd_nccl_unique_id) and travel by any side channel
int slabcomm_nccl_unique_id(void* out128);
SlabComm* slabcomm_create_nccl(int nranks, int rank, int lo, int hi, const void* uid_reduce,
                               const void* uid_halo, int* err);
SlabComm* slabcomm_create_host(int nranks, int rank, int lo, int hi, HostAllreduceFn ar,
                               HostExchangeFn ex, void* user);
void slabcomm_destroy(SlabComm* c);

int slabcomm_nranks(const SlabComm* c);
int slabcomm_rank(const SlabComm* c);
bool slabcomm_is_host(const SlabComm* c);

// in place on the device buffer, ordered on stream s (host mode: synchronous)
int slabcomm_allreduce(SlabComm* c, double* buf, int n, int op, cudaStream_t s);
// grouped {SUM over buf[0:n_sum], MAX over buf[n_sum:n_sum + n_max]} (one NCCL group)
int slabcomm_allreduce_sum_max(SlabComm* c, double* buf, int n_sum, int n_max, cudaStream_t s);
// send[2][n_side] (side 0: rows {0,1}, side 1: rows {nx-2,nx-1}) -> recv[2][n_side]
// (side 0: the lo neighbour's top rows, side 1: the hi neighbour's bottom rows), on stream s
int slabcomm_exchange(SlabComm* c, const double* send, double* recv, long long n_side, cudaStream_t s);

}  // namespace emhd
