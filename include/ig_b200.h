/*
 * ig_b200.h — C-ABI of the B200-native Interpretable-Generalization hot path.
 *
 * This is the drop-in boundary of SURVEY.md §8(b).  Every entry point takes
 * plain pointers and sizes (no torch / C++ types) and returns an int status.
 * Packed rows use the reference layout exactly (proj/include/ig/bitpack.hpp:15-26,
 * proj/src/bitpack.cpp:17-28): row-major n x K int64 words, K = ceil(L/64),
 * bit j in word j/64 at position j%64 (LSB first), padding bits >= L zero.
 *
 * Host pointers are the default.  Functions suffixed `_device` take device
 * pointers that stay resident in HBM (the bench's `value` leg); everything
 * runs on the context's stream (ig_ctx_set_stream).
 *
 * Each declaration cites the reference interface it replaces.  A thin C++
 * shim that implements `ig::KernelBackend` and the `mine.hpp` free functions on
 * top of this ABI is shown in INTEGRATION.md.
 */
#ifndef IG_B200_H
#define IG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status
 * One code per reference exception type; no exception crosses the ABI.      */
enum ig_status {
    IG_OK = 0,
    IG_E_INVALID_ARG = 1, /* std::invalid_argument  kernels.cpp:22-36,93,110; bitpack.cpp:53-58 */
    IG_E_RANGE = 2,       /* std::out_of_range      bitpack.cpp:20-24 */
    IG_E_CONFIG = 3,      /* ig::ConfigError        kernels.cpp:12-15,193; pipeline.cpp:113-119 */
    IG_E_IO = 4,          /* ig::IoError            csv.cpp:98-103 */
    IG_E_DATA = 5,        /* ig::DataError          csv.cpp:32-36; pipeline.cpp:42,110,174,190,310,317 */
    IG_E_OVERFLOW = 6,    /* ig::ArithmeticError    kernels.cpp:40-46,174-176; mine.hpp:46-51 */
    IG_E_CUDA = 7,        /* CUDA runtime failure (no reference counterpart) */
    IG_E_NCCL = 8,
    IG_E_OOM = 9
};

typedef struct ig_ctx ig_ctx;

/* Context = one device + its streams + the resident buffers.  Calls on one
 * context from several threads are safe and serialised (a per-context lock);
 * callers that want them to run concurrently use one context per thread
 * (kernels.hpp:23-26: backend methods are pure and may be called
 * concurrently; every call is a pure function of its inputs).  Result objects
 * (models, encodings, candidate sets) may be read from several threads. */
int ig_ctx_create(int device, ig_ctx** out);
void ig_ctx_destroy(ig_ctx* ctx);
/* Message of the calling thread's last failing call (on any context; ctx is
 * accepted for symmetry and ignored). */
const char* ig_last_error(const ig_ctx* ctx);
/* Run subsequent work on `stream` (a cudaStream_t); NULL restores the context's own. */
int ig_ctx_set_stream(ig_ctx* ctx, void* stream);
/* Number of kernels this context has launched so far (bench `gpu_launches`). */
uint64_t ig_ctx_launch_count(const ig_ctx* ctx);
const char* ig_version(void);
/* Diagnostics for the bench roofline (off by default; when on, the two
 * classes run one after the other and every hot kernel launch is timed with
 * CUDA events on its stream and followed by a counting re-run, so the timed
 * path is untouched when off).  Per kernel since the last
 * ig_ctx_set_diagnostics: event time, exact useful 64-bit word-ANDs, launches.
 * kernel: 0 pair_enum (kernels 2+3: pairs x K), 1 support scan (kernel 5),
 * 2 coverage scan (kernel 4), 3 matcher (kernel 6); posting word-ANDs of live
 * list words, early exits honoured. */
int ig_ctx_set_diagnostics(ig_ctx* ctx, int on);
int ig_ctx_diag_kernel(ig_ctx* ctx, int kernel, double* kernel_ms, uint64_t* word_ands, uint64_t* launches);
/* Integer-pipe micro-benchmark: sustained LOP3.32/s and POPC.32/s of the whole
 * device (roofline denominator of the AND/POPC kernels). */
int ig_measure_int_peaks(ig_ctx* ctx, double* lop3_per_s, double* popc_per_s);

/* KernelConfig (kernels.hpp:14-21).  pair_batch / coverage_block must be >= 1
 * (kernels.cpp:12-15) and never change results; threads is ignored. */
typedef struct {
    size_t pair_batch;
    size_t coverage_block;
    size_t memory_budget_bytes;
    int threads;
} ig_kernel_config;
void ig_kernel_config_default(ig_kernel_config* cfg);

/* ---------------------------------------------------------------- KernelBackend
 * kernels.hpp:27-53 — the three batched primitives.                          */

/* out[t] = rows[left] & rows[j_begin+t]; window must lie in (left, n]
 * (kernels.hpp:33-39; kernels.cpp:19-32).  Contract conformance only: the fit
 * never crosses the boundary per left row. */
int ig_pair_intersect_batch(ig_ctx* ctx, const int64_t* rows, size_t n_rows, uint32_t logical_len,
                            size_t left, size_t j_begin, size_t j_end, int64_t* out);

/* mask[p] = 1 iff some opponent row is a superset of pattern p
 * (kernels.hpp:41-46; kernels.cpp:59-65,89-103).  coverage_block >= 1. */
int ig_coverage_any(ig_ctx* ctx, const int64_t* patterns, size_t n_patterns, uint32_t patterns_len,
                    const int64_t* opponents, size_t n_opponents, uint32_t opponents_len,
                    size_t coverage_block, uint8_t* mask);

/* out[t] = sum_p scores[p] * [pattern p subset of test t], checked int64 in
 * pattern order (kernels.hpp:48-52; kernels.cpp:40-46,67-77,105-118). */
int ig_fused_score(ig_ctx* ctx, const int64_t* patterns, size_t n_patterns, uint32_t patterns_len,
                   const int64_t* scores, size_t n_scores, const int64_t* tests, size_t n_tests,
                   uint32_t tests_len, int64_t* out);

/* ---------------------------------------------------------------- mine
 * mine.hpp:12-53.  A candidate set lives on the device; copy out on demand.   */
typedef struct ig_candidates ig_candidates;
typedef void (*ig_progress_fn)(uint64_t pairs_done, uint64_t pairs_total, uint64_t candidates_found,
                               void* user);

/* {rows[i] & rows[j] : i<j, non-empty} U {rows[i]} deduplicated by content, in
 * canonical words::less order (mine.hpp:35-40).
 * Progress (mine.hpp:31-33) is reported from the calling thread while the
 * kernel runs: pairs_done / pairs_total count the pairs (u <= v) of the
 * distinct rows the device enumerates (identical rows collapse first),
 * candidates_found the distinct candidates so far; the last call is
 * (pairs_total, pairs_total, final count). */
int ig_enumerate_candidates(ig_ctx* ctx, const int64_t* rows, size_t n_rows, uint32_t logical_len,
                            const ig_kernel_config* cfg, ig_progress_fn progress, void* user,
                            ig_candidates** out);
/* support[p] = #{i : pattern p subset of rows[i]} (mine.hpp:42-44). */
int ig_count_support(ig_ctx* ctx, ig_candidates* cands, const int64_t* rows, size_t n_rows,
                     uint32_t logical_len, const ig_kernel_config* cfg);
/* Same on plain host arrays (patterns not produced by ig_enumerate_candidates). */
int ig_count_support_rows(ig_ctx* ctx, const int64_t* patterns, size_t n_patterns, uint32_t patterns_len,
                          const int64_t* rows, size_t n_rows, uint32_t rows_len, int64_t* support);
/* score = support * size^2, checked (mine.hpp:46-48). */
int ig_score_patterns(ig_ctx* ctx, ig_candidates* cands);
/* checked sum (mine.hpp:50-51). Host-only arithmetic. */
int ig_total_score(const int64_t* scores, size_t n, int64_t* out);
size_t ig_candidates_count(const ig_candidates* c);
uint32_t ig_candidates_logical_len(const ig_candidates* c);
/* Any output pointer may be NULL; supports/scores must have been computed if requested. */
int ig_candidates_copy(ig_ctx* ctx, const ig_candidates* c, int64_t* words, int64_t* supports,
                       int64_t* scores);
void ig_candidates_free(ig_candidates* c);

/* ---------------------------------------------------------------- purify / fit
 * The coarse entry point: SPEC.md cmd_train's mining half with both
 * classes resident: enumerate -> support -> score -> total -> reject_covered
 * for attack and normal.  Dictionaries keep canonical order.     */
typedef struct ig_model ig_model;

int ig_fit(ig_ctx* ctx, const int64_t* attack, size_t n_attack, const int64_t* normal,
           size_t n_normal, uint32_t logical_len, const ig_kernel_config* cfg, ig_model** out);
int ig_fit_device(ig_ctx* ctx, const int64_t* d_attack, size_t n_attack, const int64_t* d_normal,
                  size_t n_normal, uint32_t logical_len, const ig_kernel_config* cfg, ig_model** out);
/* cls: 0 attack, 1 normal.  which: 0 candidates B^c, 1 pure dictionary P^c. */
size_t ig_model_count(const ig_model* m, int cls, int which);
uint32_t ig_model_logical_len(const ig_model* m);
int ig_model_copy(ig_ctx* ctx, const ig_model* m, int cls, int which, int64_t* words,
                  int64_t* supports, int64_t* scores);
/* Page-locked host storage for results (the reference returns its dictionaries
 * as host std::vectors, mine.hpp:13-29).  Blocks are cached
 * by size, so repeated fits reuse them: cudaHostAlloc costs ~0.1 ms/MB, and a
 * pageable device-to-host copy into fresh pages runs at a few GB/s against
 * ~55 GB/s into page-locked memory.  IG_E_OOM when the host cannot pin.     */
int ig_host_alloc(size_t bytes, void** out);
void ig_host_free(void* p);
/* Phase timings of the last fit in ms: [rows, enumerate, support, purify, order, total]. */
int ig_model_phase_ms(const ig_model* m, double* ms6);
void ig_model_free(ig_model* m);

/* evidence_scores: A = fused_score(P+, S+, T), N likewise.  */
int ig_evidence(ig_ctx* ctx, const ig_model* m, const int64_t* tests, size_t n_tests,
                uint32_t tests_len, int64_t* A, int64_t* N);
int ig_evidence_device(ig_ctx* ctx, const ig_model* m, const int64_t* d_tests, size_t n_tests,
                       uint32_t tests_len, int64_t* d_A, int64_t* d_N);

/* ---------------------------------------------------------------- pipeline
 * Kernel (1): tokenise -> vocabulary -> anti-contradiction -> pack
 * (pipeline.hpp:60-113; pipeline.cpp:171-339).  The host keeps CSV parsing,
 * schema statistics and the byte-order vocabulary sort (SURVEY.md §7 hard part 3);
 * the device computes every cell's z-score units llround(((v-mean)/std)*10^p)
 * in IEEE double, the distinct tokens, the bit lookup and the packed rows.   */
typedef struct ig_table ig_table;   /* parsed CSV (csv.hpp:9-21) */
typedef struct ig_schema ig_schema; /* DatasetSchema (pipeline.hpp:24-36) */
typedef struct ig_columns ig_columns; /* typed column arrays of a table under a schema */
typedef struct ig_encoding ig_encoding; /* vocabulary + packed rows (device resident) */

int ig_read_csv(const char* bytes, size_t len, ig_table** out);        /* csv.hpp:19 */
size_t ig_table_rows(const ig_table* t);
size_t ig_table_cols(const ig_table* t);
/* rows [begin, end) as a new table (positional split). */
int ig_table_slice(const ig_table* t, size_t begin, size_t end, ig_table** out);
void ig_table_free(ig_table* t);

/* pipeline.hpp:70-72.  attack_values / normal_values: comma-separated or NULL. */
int ig_infer_schema(const ig_table* t, const char* label_column, const char* attack_values,
                    const char* normal_values, int decimals, ig_schema** out);
int ig_schema_column(const ig_schema* s, size_t j, int* kind, double* mean, double* stddev);
size_t ig_schema_label_index(const ig_schema* s);
size_t ig_schema_cols(const ig_schema* s);
void ig_schema_free(ig_schema* s);

/* Host parse of a table under a schema into typed arrays (the "parsed
 * columns" the timed fit starts from).  Numeric cells become
 * doubles (NaN = empty cell), categorical cells interned ids (-1 = empty);
 * unparsable numeric cells -> IG_E_DATA (pipeline.cpp:188-193). */
int ig_columns_build(const ig_table* t, const ig_schema* s, int with_labels, ig_columns** out);
/* Keep a copy of the columns resident on the context's device; later encodes
 * of these columns read HBM instead of host memory (bench `value` leg). */
int ig_columns_upload(ig_ctx* ctx, ig_columns* c);
/* Start the host->device copy of the columns on the context's copy stream and
 * return at once; the next encode of these columns waits for it (one-shot).
 * Lets a caller overlap the test columns' transfer with the fit. */
int ig_columns_prefetch(ig_ctx* ctx, ig_columns* c);
/* Device CSV ingest (replaces read_csv csv.cpp:14-89,
 * split_by_ratio SPEC.md:508-516, infer_schema pipeline.cpp:107-169 and the
 * cell parsing of tokenize_row pipeline.cpp:171-202): CSV bytes -> schema + typed
 * train/test columns resident on the context's device, identical to
 * ig_read_csv -> slice (first train_rows records, or ratio_k tenths when
 * train_rows < 0) -> ig_infer_schema (training rows) -> ig_columns_build +
 * ig_columns_upload.  Records, numbers (from_chars-exact fast path, host for
 * the rest), sequential-sum statistics and first-appearance categorical ids are
 * computed on the device; quoted input takes the host reader.  *test is an
 * empty table when every record trains. */
int ig_ingest_csv(ig_ctx* ctx, const char* bytes, size_t len, const char* label_column, const char* attack_values,
                  const char* normal_values, int decimals, long long train_rows, int ratio_k, ig_schema** schema,
                  ig_columns** train, ig_columns** test);
size_t ig_columns_rows(const ig_columns* c);
/* Bytes a host->device copy of the columns moves: the numeric block in its
 * narrow exact form (per column the first decimal scale whose integer codes
 * reproduce every parsed double bitwise under IEEE division, in the smallest
 * integer type; else the raw doubles; built by ig_columns_build), the
 * categorical ids and the labels. */
size_t ig_columns_bytes(const ig_columns* c);
void ig_columns_free(ig_columns* c);

/* encode_training (pipeline.hpp:103; pipeline.cpp:273-328). */
int ig_encode_training(ig_ctx* ctx, const ig_columns* cols, ig_encoding** out);
/* encode_rows (pipeline.hpp:108-109; pipeline.cpp:330-339): test rows under
 * the training vocabulary; unseen tokens dropped. */
int ig_encode_rows(ig_ctx* ctx, const ig_columns* cols, const ig_encoding* train, ig_encoding** out);
uint32_t ig_encoding_logical_len(const ig_encoding* e);
/* which: 0 attack, 1 normal (training); 2 all rows (test encode). */
size_t ig_encoding_rows(const ig_encoding* e, int which);
const int64_t* ig_encoding_device_rows(const ig_encoding* e, int which);
int ig_encoding_copy_rows(ig_ctx* ctx, const ig_encoding* e, int which, int64_t* out);
/* Vocabulary as '\n'-terminated tokens in bit order (pipeline.hpp:40-58). */
const char* ig_encoding_vocabulary(const ig_encoding* e);
/* Anti-contradiction report (pipeline.hpp:88-100): removed source rows ascending. */
size_t ig_encoding_removed_count(const ig_encoding* e);
int ig_encoding_removed_rows(const ig_encoding* e, uint64_t* rows);
void ig_encoding_free(ig_encoding* e);

/* Fit / evidence directly on resident encodings (no host round trip). */
int ig_fit_encoded(ig_ctx* ctx, const ig_encoding* train, const ig_kernel_config* cfg, ig_model** out);
int ig_evidence_encoded(ig_ctx* ctx, const ig_model* m, const ig_encoding* tests, int64_t* A,
                        int64_t* N);
/* evidence_scores with device outputs d_A / d_N (int64[rows]), ordered on the context
 * stream.  A test encoding made by ig_encode_rows from resident or prefetched
 * columns is packed and indexed (row postings) in the background on the
 * context's index stream, overlapping a fit issued meanwhile; evidence and every
 * accessor wait for it. */
int ig_evidence_encoded_device(ig_ctx* ctx, const ig_model* m, const ig_encoding* tests, int64_t* d_A,
                               int64_t* d_N);
/* fit (mine.hpp:38-51 + reject_covered) and evidence_scores
 * of a test encoding in one call — the train-and-score of the reference's
 * pipeline: each class's matcher starts as soon as that class's pure
 * dictionary is ready, overlapping the other class's fit.  Results identical to
 * ig_fit_encoded + ig_evidence_encoded(_device).  _host writes A / N to host
 * memory. */
int ig_fit_evidence_encoded(ig_ctx* ctx, const ig_encoding* train, const ig_encoding* tests,
                            const ig_kernel_config* cfg, ig_model** out, int64_t* d_A, int64_t* d_N);
int ig_fit_evidence_encoded_host(ig_ctx* ctx, const ig_encoding* train, const ig_encoding* tests,
                                 const ig_kernel_config* cfg, ig_model** out, int64_t* A, int64_t* N);

/* ---------------------------------------------------------------- infer (host arithmetic)
 * SPEC.md:434-452 (spec-only in the reference).  fit_normal_stats: mean and
 * population std of the strictly positive N (batch fit); fewer than
 * two -> (0, 0).  classify: R2 A=N=0 -> attack (reg 3), R1 A>=N -> attack
 * (reg 1), R3 N < mu - r*sigma -> attack (reg 4), else normal (reg 2).  The
 * squared deviations and the R3 threshold round as single FMAs, as the
 * reference's -march=native build (proj/CMakeLists.txt:10-18) contracts them.
 * label / regulation may be NULL.                                          */
int ig_fit_normal_stats(const int64_t* n_vals, size_t n, double* mu, double* sigma);
int ig_classify(const int64_t* A, const int64_t* N, size_t n, double mu, double sigma, double r, uint8_t* label,
                uint8_t* regulation);

/* ---------------------------------------------------------------- archive / explain
 * SURVEY.md §8(f) ranks 1-2.  ModelArchive: schema
 * text with exact hex-float statistics + vocabulary in bit order + the pure
 * dictionaries; an encoding rebuilt from (schema, vocabulary) tokenises test
 * rows exactly like the training encoding.                                  */
/* *len = text size; copies min(cap-1, len) bytes + NUL when buf is given. */
int ig_schema_to_text(const ig_schema* s, char* buf, size_t cap, size_t* len);
int ig_schema_from_text(const char* text, ig_schema** out);
/* vocab: '\n'-terminated tokens in bit order (ig_encoding_vocabulary). */
int ig_encoding_from_vocabulary(const ig_schema* s, const char* vocab, ig_encoding** out);
/* Pure dictionaries (canonical order) -> model usable by ig_evidence* / ig_explain. */
int ig_model_from_dictionaries(ig_ctx* ctx, uint32_t logical_len, const int64_t* words_attack,
                               const int64_t* supports_attack, const int64_t* scores_attack, size_t n_attack,
                               const int64_t* words_normal, const int64_t* supports_normal,
                               const int64_t* scores_normal, size_t n_normal, ig_model** out);
/* ModelArchive writer / reader (SPEC.md:568-573 fields, :607 round trip,
 * :611 format): format_version, tool version, provenance (free text the caller
 * supplies: input digest, timestamps, ...), classifier parameters (r, stats mode
 * "batch" = mu_N / sigma_N fitted per predict batch, or "frozen" with the
 * values), the schema (exact hex-float statistics), the vocabulary in bit
 * order and both pure dictionaries (canonical order, packed words + supports +
 * scores as base-64 sections).  save -> load -> save is byte-identical.
 * ig_model_save: *len = archive size; copies min(cap-1, len) bytes + NUL when
 * buf is given (call with buf = NULL first to size it).  vocabulary: the
 * '\n'-terminated tokens in bit order (ig_encoding_vocabulary).
 * ig_model_load: a model usable by ig_evidence* / ig_explain, its schema and
 * an encoding that tokenises test rows exactly like the training encoding
 * (ig_encode_rows); params->provenance is set to NULL, the text is copied to
 * `provenance` (prov_len = its length). */
typedef struct {
    double r;              /* R3 parameter (default 0.568) */
    int stats_frozen;      /* 0: batch statistics; 1: mu / sigma below */
    double mu, sigma;
    const char* provenance; /* NUL-terminated; NULL = empty */
} ig_archive_params;
int ig_model_save(ig_ctx* ctx, const ig_model* m, const ig_schema* schema, const char* vocabulary,
                  const ig_archive_params* params, char* buf, size_t cap, size_t* len);
int ig_model_load(ig_ctx* ctx, const char* data, size_t n_bytes, ig_model** model, ig_schema** schema,
                  ig_encoding** encoding, ig_archive_params* params, char* provenance, size_t prov_cap,
                  size_t* prov_len);

/* explain: indices into P^cls (ascending) of the patterns
 * contained in one test row; *n_found may exceed cap (call again larger). */
int ig_explain(ig_ctx* ctx, const ig_model* m, int cls, const int64_t* row, uint32_t logical_len, uint32_t* idx,
               size_t cap, size_t* n_found);

/* ---------------------------------------------------------------- multi-GPU
 * SURVEY.md §8(e).  One shard per rank (one process per GPU); training rows
 * are replicated (every rank runs ig_encode_training on the same columns).
 * Per class: ig_shard_enumerate dedups the pairs of this rank's tiles
 * (round-robin over the u <= v tile triangle of the distinct canonical rows)
 * and buckets the distinct candidates by owner (content fingerprint mod
 * world) as 8-byte (u, v) row-pair records; the caller exchanges them
 * (all-to-all, e.g. NCCL over NVLink) and hands each rank what it received to
 * ig_shard_receive, which dedups exactly across ranks.  ig_shard_finish runs
 * support / score / coverage / order on the owned candidates; its partial
 * totals must be summed across ranks and checked <= INT64_MAX (mine.hpp:50-51).
 * Evidence of the owned dictionaries (ig_evidence* on ig_shard_model) are
 * partial sums; their sum over ranks is the full A / N.                    */
typedef struct ig_shard ig_shard;
int ig_shard_create(ig_ctx* ctx, const ig_encoding* train, int rank, int world, const ig_kernel_config* cfg,
                    ig_shard** out);
int ig_shard_enumerate(ig_ctx* ctx, ig_shard* s, int cls, uint64_t* counts, const void** d_send);
int ig_shard_receive(ig_ctx* ctx, ig_shard* s, int cls, const void* d_recv, uint64_t n_records);
int ig_shard_finish(ig_ctx* ctx, ig_shard* s, uint64_t* partial_totals);
const ig_model* ig_shard_model(const ig_shard* s);
void ig_shard_free(ig_shard* s);

#ifdef __cplusplus
}
#endif
#endif /* IG_B200_H */
