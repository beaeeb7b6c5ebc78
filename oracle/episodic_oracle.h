/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") of the reference's
 * counting algorithm, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER. The product library never links it.
 *
 * Episode batches use the same CSR layout as the product C-ABI
 * (include/episodic_b200.h): off[n_eps+1] node offsets into types[]; the
 * constraints of episode e live at lo/hi[off[e]-e .. off[e+1]-e-1).
 *
 * Parity pinning: every function here is checked against the reference's own
 * known-answer tests and against the reference compiled in place
 * (oracle/_ref) through the committed fixtures in tests/golden/.
 */
#ifndef EPISODIC_ORACLE_H
#define EPISODIC_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 0 ok, 1 invalid argument, 2 data error (messages as the reference's). */
int orc_validate_stream(const uint32_t* types, const int64_t* times, uint64_t n,
                        uint32_t alphabet, char* msg, size_t msg_len);

/* count_fsm restated (E/fsm.hpp:45-106). Returns UINT64_MAX on an invalid
 * episode (validate, E/types.hpp:82-92). */
uint64_t orc_count_fsm(const uint32_t* types, const int64_t* times, uint64_t n,
                       const uint32_t* ep_types, const int64_t* lo, const int64_t* hi,
                       uint32_t n_nodes);

/* oracle_count restated (E/oracle.hpp:21-85): exhaustive enumeration of
 * occurrence intervals + greedy max non-overlap. Returns UINT64_MAX when the
 * enumeration bound (500 events, 6 nodes, E/oracle.hpp:14-17) is exceeded. */
uint64_t orc_oracle_count(const uint32_t* types, const int64_t* times, uint64_t n,
                          const uint32_t* ep_types, const int64_t* lo, const int64_t* hi,
                          uint32_t n_nodes);

/* Greedy max non-overlap over intervals (E/oracle.hpp:65-79). */
uint64_t orc_max_nonoverlap(const int64_t* starts, const int64_t* ends, uint64_t n);

/* Batch count_fsm over a CSR episode batch with `threads` POSIX threads
 * (episode-parallel, like E/miner.hpp:146-150). Returns 0 or 1 (invalid). */
int orc_count_batch(const uint32_t* types, const int64_t* times, uint64_t n,
                    const uint32_t* off, const uint32_t* ep_types, const int64_t* lo,
                    const int64_t* hi, uint64_t n_eps, unsigned threads, uint64_t* out);

/* Stream digest used by the golden fixtures (oracle/make_golden.cpp). */
uint64_t orc_fnv_stream(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet);

#ifdef __cplusplus
}
#endif
#endif
