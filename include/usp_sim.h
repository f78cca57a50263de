/* usp_sim.h — the reference's public C ABI, served by the B200 engine.
 *
 * ABI-identical to the reference's include/uspsim.h:19-55 (same function
 * names, argument meaning, status numbering and ownership rules), exported
 * by libusp_b200.so, so a program or binding written against libuspsim
 * links against the B200 library unchanged:
 *
 *   {"command": "simulate", "params": {batch, seqlen, heads, kv_heads,
 *    head_size, ulysses, ring, causal, precision, seed, check, tolerance}}
 *
 * runs the reference's `simulate` (src/api/commands.cpp:85-282): inputs
 * from UniformSource(seed) in [-1, 1) filling Q, K, V, dO (commands.cpp:
 * 90-102), every rank of the ulysses x ring mesh runs usp_attn_fwd then
 * usp_attn_bwd on the GPU (one host thread per rank over the in-process
 * transport, the analogue of simcomm::World::run), and with "check": true
 * the gathered O, dQ, dK, dV are compared with an fp64 single-device
 * reference on the same (bf16-rounded) inputs, computed on the GPU.
 *
 * Differences, by design:
 *   * precision is "bf16" (the engine's bf16-in / fp32-accumulate path,
 *     the default); "fp32" / "fp64" are rejected as invalid input (they are
 *     the CPU library's precisions). Default tolerance 2e-2 (max-abs, the
 *     reference's check metric);
 *   * the ledger carries the collectives the engine executes: the position
 *     all_gathers of the reference (usp_attention.cpp:53,
 *     ring_attention.cpp:56,95) are static on B200 and absent; every other
 *     event keeps the reference's (group, step) numbering and bytes as moved
 *     (bf16, fp32 for the circulating dK/dV partials);
 *   * optional param "device" (CUDA ordinal, default 0) hosts all ranks;
 *   * "balance" is served (host arithmetic over the zigzag layout);
 *     "cost" and "plan" (analytic, host-only, outside the
 *     accelerated path) return an invalid-input report naming the
 *     reference library.
 */
#ifndef USP_SIM_H
#define USP_SIM_H

#include "usp_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum uspsim_status {
  USPSIM_OK = 0,
  USPSIM_TOLERANCE_EXCEEDED = 1,
  USPSIM_INVALID_INPUT = 2,
  USPSIM_INTERNAL_ERROR = 3,
} uspsim_status;

typedef struct uspsim_report uspsim_report;

/* uspsim.h:33-40 */
USP_API uspsim_status uspsim_run(const char* request_json, uspsim_report** out_report);
/* uspsim.h:42-49 */
USP_API const char* uspsim_report_json(const uspsim_report* report);
USP_API const char* uspsim_report_text(const uspsim_report* report);
USP_API const char* uspsim_report_ledger_csv(const uspsim_report* report);
USP_API int uspsim_report_exit_code(const uspsim_report* report);
USP_API void uspsim_report_free(uspsim_report* report);
/* uspsim.h:51-54 */
USP_API const char* uspsim_last_error(void);
USP_API const char* uspsim_version(void);

#ifdef __cplusplus
}
#endif

#endif /* USP_SIM_H */
