/* usp_oracle.h — CPU restatement of the reference's USP attention forward.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the B200 engine:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it. The product path (paper_2405_07719_b200) never
 * links, imports or calls anything in oracle/.
 *
 * Every function restates one reference routine (file:line into
 * /root/reference/proj) with the same loop order and the same floating-point
 * operation sequence, so that on identical fp64 inputs it reproduces the
 * reference bit for bit (pinned by tests/test_oracle.py against oracle/_ref,
 * the reference's own sources compiled by oracle/Makefile, and against the
 * committed golden vectors in tests/golden/).
 *
 * Layouts follow the reference Tensor4 (src/numerics/tensor.hpp:66-68):
 * row-major (batch, seq, heads, head_size).
 */
#ifndef USP_ORACLE_H
#define USP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* UniformSource (src/common/random.hpp:15-29): mt19937_64, top 53 bits,
 * mapped to [lo, hi). Writes n consecutive draws of one stream seeded with
 * `seed`. The reference fills Q, K, V, dO from one stream in that order
 * (src/api/commands.cpp:90-102, tests/usp_harness.hpp:30-41). */
void uo_uniform_stream(uint64_t seed, double lo, double hi, int64_t n,
                       double* out);

/* reference_attention<double> (src/numerics/attention.cpp:51-93).
 * positions == NULL means storage order (attention.cpp:38-40). Returns 0 or
 * a negative error code for shape errors (attention.cpp:15-36). */
int uo_reference_attention(const double* q, const double* k, const double* v,
                           int64_t batch, int64_t seq, int64_t heads,
                           int64_t kv_heads, int64_t head_size, int causal,
                           const int64_t* positions, double* out);

/* SoftmaxState<double> (attention.cpp:172-264) driven as one update over a
 * query subset: rows q (batch, q_len, heads, hs) at original positions q_pos
 * against keys k/v (batch, k_len, kv_heads, hs) at k_pos, with the
 * BlockMask::causal semantics of attention.hpp:32-34. Produces finalize()
 * (attention.cpp:232-254) into out and logsumexp() (attention.cpp:256-264,
 * natural log, (b*q_len+t)*heads+h) into lse. A row that saw no key gets
 * out = NaN and lse = -inf (the reference throws "saw no keys"); the return
 * value is the number of such rows. */
int64_t uo_softmax_rows(const double* q, const double* k, const double* v,
                        int64_t batch, int64_t q_len, int64_t k_len,
                        int64_t heads, int64_t kv_heads, int64_t head_size,
                        int causal, const int64_t* q_pos, const int64_t* k_pos,
                        double* out, double* lse);

/* zigzag_partition (src/usp/partition.cpp:12-33): out[R][L/R].
 * Returns -1 (kConstraint) when L % (2R) != 0. */
int uo_zigzag_partition(int64_t seq_len, int ring, int64_t* out);
/* even_partition (partition.cpp:35-50). Returns -1 when L % R != 0. */
int uo_even_partition(int64_t seq_len, int ring, int64_t* out);
/* causal_pair_counts (partition.cpp:52-72) over an R x (L/R) assignment. */
int uo_causal_pair_counts(const int64_t* assignment, int ring,
                          int64_t seq_len, int64_t* counts);
/* ShardSpec::positions_for (partition.cpp:74-105) with the ProcessMesh rank
 * map rank = r*U + u (src/simcomm/mesh.cpp:23-39). Returns -1 on the
 * constraint violations of partition.cpp:78-92. */
int uo_positions_for(int ulysses, int ring, int64_t seq_len, int zigzag,
                     int rank, int64_t* out);

/* usp_attention<double> forward (src/usp/usp_attention.cpp:43-65) for every
 * rank of a U x R mesh, simulated in one thread. Inputs are the GLOBAL
 * tensors in original token order; the emulation shards them with
 * positions_for, applies the Ulysses all-to-all layout
 * (src/usp/all_to_all_4d.cpp:13-59), runs ring_attention's step order
 * (src/usp/ring_attention.cpp:45-76: step t folds the K/V block of ring
 * source (my - t) mod R into a SoftmaxState) and the inverse all-to-all
 * (all_to_all_4d.cpp:62-107).
 *   out_global: (batch, L, heads, hs) reassembled with place_rows
 *               (partition.hpp:75-87);
 *   lse: U*R consecutive blocks, rank-major, each the head-sharded
 *        logsumexp (batch, L/R, heads/U) in head_positions order.
 * Returns 0, or -1 on a constraint violation (usp_attention.cpp:15-38). */
int uo_usp_forward(const double* q, const double* k, const double* v,
                   int64_t batch, int64_t seq, int64_t heads, int64_t kv_heads,
                   int64_t head_size, int ulysses, int ring, int causal,
                   double* out_global, double* lse);

/* reference_attention_grad<double> (attention.cpp:95-170). */
int uo_reference_attention_grad(const double* q, const double* k, const double* v,
                                const double* dout, int64_t batch, int64_t seq,
                                int64_t heads, int64_t kv_heads, int64_t head_size,
                                int causal, const int64_t* positions, double* dq,
                                double* dk, double* dv);

/* usp_attention_backward<double> (usp_attention.cpp:68-89,
 * ring_attention.cpp:79-155, attention.cpp:266-324) after the forward, over
 * every rank of a U x R mesh; global dq, dk, dv in original token order. */
int uo_usp_backward(const double* q, const double* k, const double* v, const double* dout,
                    int64_t batch, int64_t seq, int64_t heads, int64_t kv_heads,
                    int64_t head_size, int ulysses, int ring, int causal, double* dq,
                    double* dk, double* dv);

#ifdef __cplusplus
}
#endif

#endif /* USP_ORACLE_H */
