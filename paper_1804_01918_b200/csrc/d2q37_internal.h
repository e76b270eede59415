// d2q37_internal.h -- declarations shared by the product's translation units.
#pragma once

#include <cstdint>
#include <string>

#include "d2q37_b200.h"

namespace d2q37 {

constexpr int kHostNpop = D2Q37_NPOP;

void build_model(d2q37_model* m);
void host_equilibrium(const d2q37_model& m, double rho, double ux, double uy, double temp, double* f_eq);
bool host_macros(const d2q37_model& m, const double* f, double out[4]);
bool host_collide_site(const d2q37_model& m, const double* f, double omega, double* out);
void philox4x32_10(const uint32_t in[4], const uint32_t key[2], uint32_t out[4]);
double philox_u01(uint64_t seed, uint64_t counter);
void make_lattice(int kind, int lx, int ly, uint64_t seed, const double* params, const d2q37_model& m,
                  double* out, int nthreads);

void set_error(const std::string& msg);

// NCCL, loaded on first multi-GPU use (d2q37_nccl.cpp).
struct NcclApi;
const NcclApi* nccl_api(std::string* why);
int nccl_unique_id(unsigned char* id, std::string* why);
// Returns an opaque ncclComm_t.
int nccl_comm_init(void** comm, int nranks, const unsigned char* id, int rank, std::string* why);
void nccl_comm_destroy(void* comm);
// One grouped exchange: send_hi -> hi_peer, recv_lo <- lo_peer, send_lo -> lo_peer,
// recv_hi <- hi_peer (peers < 0 are skipped).  count doubles per message.
int nccl_exchange(void* comm, void* stream, const double* send_lo, double* recv_lo, int lo_peer,
                  const double* send_hi, double* recv_hi, int hi_peer, size_t count, std::string* why);

}  // namespace d2q37
