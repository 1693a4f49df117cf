/* Fused expert-parallel exchange on the NCCL device API (PAPER:648-671
 * "Expert Parallelism ... token distribution and gradient aggregation").
 *
 * The host-API exchange (include/omnimoe.h omnimoe_ep_pack / _unpack / _combine +
 * torch.distributed all_to_all) moves the dispatch and return messages with
 * NCCL collectives.  This library moves the same bytes with the GPU's own stores over
 * NVLink / NVSwitch into symmetric memory windows of the peers (ncclMemAlloc +
 * ncclCommWindowRegister, pointers from ncclGetLsaPointer), ordered by in-kernel LSA
 * barriers: no NCCL collective and no host involvement between the pack kernel and the
 * receiver's schedule.  Layouts are those of omnimoe_ep_pack, so the receiver runs the
 * same unpack / schedule / expert_fwd, and the home rank the same combine.
 *
 * Separate library (libomnimoe_ep.so, links libnccl): libomnimoe.so stays NCCL-free.
 * One communicator per process (rank), single node (the LSA team is the world).
 * All pointers are device pointers unless stated; calls enqueue on `stream` and return
 * OMNIMOE_* status codes (include/omnimoe.h), with text in omnimoe_ep_last_error(). */
#ifndef OMNIMOE_EP_H_
#define OMNIMOE_EP_H_
#include <stddef.h>
#include <stdint.h>

#include "omnimoe.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct omnimoe_ep_comm omnimoe_ep_comm;

/* Size of the NCCL unique id (bytes) and its creation on one rank (host memory out);
 * the caller broadcasts it (e.g. torch.distributed) before omnimoe_ep_dev_create. */
size_t omnimoe_ep_dev_unique_id_bytes(void);
omnimoe_status omnimoe_ep_dev_unique_id(void* out);

/* Collective over the `world` ranks: communicator, device communicator (LSA barriers)
 * and four symmetric windows sized for
 *   counts  int64 [world][world][2]   counts[src][dst] = (rows, records) src sends dst
 *   x_recv  bf16  [row_cap][d]        the x rows this rank receives, by source rank
 *   rec     int32 [rec_cap][3]        its task records (local id, gate bits, ROW index)
 *   y_ret   bf16  [row_cap][d]        the partial rows it gets back, by destination
 * row_cap >= rows any rank receives (<= the global batch), rec_cap >= records. */
omnimoe_status omnimoe_ep_dev_create(const void* unique_id, int32_t rank, int32_t world, int64_t d,
                                     int64_t row_cap, int64_t rec_cap, omnimoe_ep_comm** out);
omnimoe_status omnimoe_ep_dev_destroy(omnimoe_ep_comm* comm);
/* This rank's windows (device pointers, valid until destroy). */
omnimoe_status omnimoe_ep_dev_buffers(const omnimoe_ep_comm* comm, void** x_recv, int32_t** rec_recv,
                                      void** y_ret, int64_t** counts);

/* Dispatch: from omnimoe_ep_pack's outputs (x_send [rows][d] and rec_send [records][3]
 * by destination, send_counts int64 [world][2]) write every rank's counts row into all
 * peers' count windows, barrier, then store each destination block at its offset in the
 * destination's x_recv / rec windows (source blocks in rank order; record slots turned
 * into the receiver's row index), barrier.  After it, x_recv / rec / counts of every
 * rank are complete (stream order). */
omnimoe_status omnimoe_ep_dev_dispatch(omnimoe_ep_comm* comm, const void* x_send, const int32_t* rec_send,
                                       const int64_t* send_counts, omnimoe_stream_t stream);
/* Return: the partial rows of the rows this rank received (bf16 [rows_recv][d], the
 * x_recv order), each stored into its home rank's y_ret window at the position of the
 * home's x_send row; barrier.  The home then runs omnimoe_ep_combine over y_ret. */
omnimoe_status omnimoe_ep_dev_return(omnimoe_ep_comm* comm, const void* y_part, int64_t rows_recv,
                                     omnimoe_stream_t stream);

const char* omnimoe_ep_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
