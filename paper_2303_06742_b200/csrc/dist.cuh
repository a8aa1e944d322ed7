// Multi-GPU plumbing (x-slab domain decomposition): transports and halo kernels.
#pragma once
#include "stgmg_internal.cuh"

namespace stgmg {

// Exchange / reduction backend.  rank q's x-neighbours are q-1 and q+1.
struct Transport {
  int rank = 0, nranks = 1;
  virtual ~Transport() {}
  virtual bool graph_capturable() const = 0;
  // send sl to the left neighbour / sr to the right one, receive rl from the left / rr from the right
  virtual int halo(const double* sl, long long nsl, const double* sr, long long nsr, double* rl, long long nrl,
                   double* rr, long long nrr, cudaStream_t s) = 0;
  virtual int allreduce_sum(double* dev, int n, cudaStream_t s) = 0;               // in place, fixed rank order
  virtual int allgather(const double* send, long long n, double* recv, cudaStream_t s) = 0;   // recv: nranks * n
};

Transport* make_nccl_transport(void* comm, int rank, int nranks);
void* loopback_hub_create(int n);
void loopback_hub_destroy(void* hub);
Transport* make_loopback_transport(void* hub, int rank);
Transport* make_shm_transport(void* comm);
int shm_comm_create(const char* name, int nranks, int rank, long long cap_doubles, void** out);
int shm_comm_destroy(void* comm);
int nccl_unique_id(unsigned char out[128]);
int nccl_comm_create(const unsigned char id[128], int nranks, int rank, void** comm);
int nccl_comm_destroy(void* comm);

long long halo_count(const LevelGeom& g, int k1, int nxq, int nxp);
cudaError_t launch_halo(const LevelGeom& g, int k1, int xq0, int nxq, int xp0, int nxp, const double* v, double* buf,
                        int unpack, cudaStream_t s);
cudaError_t launch_owned_mask(const LevelGeom& g, int q0, int q1, int p0, int p1, unsigned char* mask, cudaStream_t s);

}  // namespace stgmg
