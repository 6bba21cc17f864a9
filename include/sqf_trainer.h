/* sqf_trainer.h — C ABI of the B200 training step, the drop-in for the
 * reference's Trainer (seqforge include/seqforge/trainer.hpp:80-125). The
 * reference is a C++ library with no FFI of its own; these entries are what a
 * binding of its Trainer would call (see INTEGRATION.md for the C++ adapter
 * and the ctypes stub). Status convention: 0 ok, 1 "data exhausted"
 * (train_one), negative = error class of the reference's taxonomy
 * (common.hpp:11-34) with the message in sqf_last_error():
 *   -1 ConfigError -2 ShapeError -3 BoundsError -4 CapacityError
 *   -5 IntegrityError -6 DivergenceError -7 RegistryError -8 IoError
 *   -10 DeviceError (CUDA/NCCL) -9 other
 */
#ifndef SQF_TRAINER_H
#define SQF_TRAINER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* StepStats (trainer.hpp:57-66) */
typedef struct sqf_step_stats {
  int64_t step;
  double loss;     /* summed over tokens, unnormalised, unscaled */
  double nll;
  int64_t ntokens;
  int64_t ncorrect;
  double lr;
  int32_t skipped; /* fp16 overflow: scaler updated, nothing else */
  int32_t _pad;
  double scale;    /* loss scale used (0 when not in fp16) */
} sqf_step_stats;

const char* sqf_last_error(void);
/* status code of the last failure on this thread (for entries returning NULL) */
int sqf_last_status(void);

/* NCCL unique id (128 bytes) for multi-process data parallelism; rank 0
 * creates it and the launcher broadcasts it (torch.distributed store). */
int sqf_nccl_unique_id(void* out128);

/* Trainer(cfg, task) (trainer.hpp:84-85, trainer.cpp:89-142).
 * arch + raw user overrides resolve like Registry::resolve_architecture
 * (registry.cpp:96-110). With npairs > 0 the in-memory corpus (eos-terminated
 * id sequences, concatenated) is the task; otherwise cfg["task"] is made
 * through the registry ("synthetic"). rank/world: this process's place in
 * the data-parallel group (world 1 = single GPU; nccl_id ignored). */
void* sqf_trainer_create(const char* arch, const char* const* keys, const char* const* vals, int n,
                         const int32_t* src_len, const int32_t* tgt_len, const int32_t* src_ids,
                         const int32_t* tgt_ids, int npairs, int src_vocab, int tgt_vocab,
                         int rank, int world, const void* nccl_id);
void sqf_trainer_free(void* t);

/* The gradient exchange between data-parallel ranks (the reference's
 * all_reduce, trainer.cpp:75-87, across processes). sqf_trainer_create uses
 * NCCL (nccl_id from sqf_nccl_unique_id). sqf_trainer_create_host_collective
 * instead hands every bucket (and the 4-double step statistics) to `fn` as a
 * pinned host copy to be summed in place over all ranks -- a test/tooling
 * backend (e.g. torch.distributed gloo) that runs the same N>1 trainer path
 * without NCCL. fn returns 0 on success. dtype codes: */
enum sqf_coll_dtype { SQF_COLL_F32 = 0, SQF_COLL_F16 = 1, SQF_COLL_BF16 = 2, SQF_COLL_F64 = 3 };
typedef int (*sqf_host_allreduce_fn)(void* buf, int64_t count, int dtype, void* user);
void* sqf_trainer_create_host_collective(const char* arch, const char* const* keys, const char* const* vals, int n,
                                         const int32_t* src_len, const int32_t* tgt_len, const int32_t* src_ids,
                                         const int32_t* tgt_ids, int npairs, int src_vocab, int tgt_vocab,
                                         int rank, int world, sqf_host_allreduce_fn fn, void* user);
/* "nccl", "host" or "none" (world 1) */
const char* sqf_trainer_collective(void* t);

/* A task made through the registry from the resolved config's "task" key
 * (Registry::make_task; "translation" = TranslationTask, tasks.cpp:7-33,
 * reading train_src/train_tgt text and dict_src/dict_tgt or building the
 * dictionaries with min_count). info gives the dictionary sizes, pair count
 * and total ids; pairs fills eos-terminated ids, concatenated. */
void* sqf_task_create(const char* arch, const char* const* keys, const char* const* vals, int n);
void sqf_task_free(void* t);
int sqf_task_info(void* t, int32_t* src_vocab, int32_t* tgt_vocab, int32_t* npairs, int64_t* src_tokens,
                  int64_t* tgt_tokens);
int sqf_task_pairs(void* t, int32_t* src_len, int32_t* tgt_len, int32_t* src_ids, int32_t* tgt_ids);

/* Trainer::train_one (trainer.cpp:204-208): 0 ok, 1 exhausted */
int sqf_trainer_train_one(void* t, sqf_step_stats* out);
/* Trainer::train_step (trainer.cpp:210-273): sub[w][a] given as corpus-index
 * member lists, counts[w*accum + a] members each, concatenated. */
int sqf_trainer_train_step(void* t, const int32_t* members, const int32_t* counts, sqf_step_stats* out);
/* Trainer::evaluate (trainer.cpp:275-289) over the trainer's own corpus
 * subset given by corpus indices (teacher-forced, fp32 master). */
int sqf_trainer_evaluate(void* t, const int32_t* corpus_idx, int n, double* loss, double* nll,
                         int64_t* ntokens, int64_t* ncorrect);

int64_t sqf_trainer_num_params(void* t);
/* fp32 master in the reference's canonical manifest order */
int sqf_trainer_params(void* t, float* out);
int sqf_trainer_set_params(void* t, const float* in); /* then rebroadcast() */
/* last step's reduced gradient (before unscale / 1/ntokens), canonical order */
int sqf_trainer_last_grads(void* t, float* out);
int sqf_trainer_manifest_size(void* t);
int sqf_trainer_manifest_entry(void* t, int i, char* name, int cap, int64_t* offset, int64_t* numel,
                               int64_t* device_offset);
int sqf_trainer_adam_state(void* t, float* m, float* v, int64_t* step_count); /* canonical order */
int sqf_trainer_scaler(void* t, double* scale, int64_t* successes);
int sqf_trainer_progress(void* t, int64_t* step, int32_t* epoch, int32_t* cursor, int32_t* nbatches);
int sqf_trainer_set_injector(void* t, const int64_t* steps, int n); /* set_overflow_injector */
int sqf_trainer_restore(void* t, int64_t step, int32_t epoch, int32_t cursor, double scale,
                        int64_t successes);
/* our kernel launches during the last train_step, and its device time (ms) */
int64_t sqf_trainer_kernel_launches(void* t);
float sqf_trainer_last_step_ms(void* t);
/* The optimizer update of a step runs on a side stream, overlapped with the
 * next step's forward (which waits per parameter range). flush: make the
 * trainer stream wait for it and return the device time (ms) from the end of
 * the last step's main-stream work to that point (timing closure). */
float sqf_trainer_flush_ms(void* t);
/* host->device bytes of the last step (returned) and device->host (*d2h) */
int64_t sqf_trainer_last_io_bytes(void* t, int64_t* d2h);
/* CUDA stream the trainer launches on (cudaStream_t) */
void* sqf_trainer_stream(void* t);
/* Checkpoints in the reference's SQFG v2 container (docs/checkpoint_format.md;
 * save_checkpoint / load_checkpoint, checkpoint.cpp:187-389). save: atomic,
 * canonical-order FP32 params and Adam moments, config with provenance,
 * scaler and epoch cursor. load: restores all of it into a trainer built with
 * the same architecture (manifest must match; IntegrityError otherwise);
 * *version = the file's format version (v1 files are upgraded). */
int sqf_trainer_save(void* t, const char* path);
int sqf_trainer_load(void* t, const char* path, int32_t* version);
/* Raw parse (read_checkpoint, checkpoint.cpp:226-320): header, table and
 * FNV-1a checksums verified. info gives the sizes; read fills params[nparams],
 * opt[nopt] and meta (sorted "key = value\n" lines, NUL-terminated). */
int sqf_checkpoint_info(const char* path, int32_t* version, int64_t* nparams, int64_t* nopt,
                        int64_t* meta_bytes);
int sqf_checkpoint_read(const char* path, float* params, float* opt, char* meta, int64_t meta_cap);

/* Data-parallel timeline model (simulate_timeline / format_report,
 * simulator.cpp:12-229): scenario text (workers, accum, mode
 * serial_sync|overlap|overlap_accum, compute rows, buckets) in, the report
 * text ("makespan", "idle <w>", "exposed_comm", "total_compute", %.17g) out. */
int sqf_simulate_timeline(const char* scenario, char* report, int cap);

/* all-reduce/backward overlap of the last step (config overlap_allreduce; with
 * world 1 only under overlap_simulate): bucket indices in issue order (up to
 * cap written), *early = how many were issued while backward was running.
 * Returns the number of buckets issued. Replaces the single post-backward
 * all_reduce of trainer.cpp:246 (all_reduce, trainer.cpp:75-87). */
int sqf_trainer_overlap_log(void* t, int32_t* order, int cap, int32_t* early);
/* per-launch CUDA-event profiling of the following steps (on = 1) and its
 * accumulated per-class totals: class 0..9 = gemm_fwd, gemm_dgrad,
 * gemm_wgrad, attn_fwd, attn_bwd, layernorm, xent, embed, bias_grad, optim.
 * Returns the class name, or NULL past the last class. */
/* on: 0 off, 1 serialised per-launch timing, 2 timeline of the concurrent
 * schedule (see sqf_trainer_timeline) */
int sqf_trainer_set_profile(void* t, int on);
/* timeline mode: launches of the last step as [stream, class, t0 ms, t1 ms]
 * relative to the step start (stream 0 main, 1 side, 2 comm); returns the
 * count (writes at most cap rows) */
int sqf_trainer_timeline(void* t, float* out, int cap);
const char* sqf_trainer_profile(void* t, int cls, double* ms, double* flops, double* bytes, int64_t* launches);

/* ---------------- host-side boundary pieces (no GPU needed) --------------- */
/* synthetic WMT-shaped corpus; two-call protocol: pass
 * null id buffers to get total lengths in *src_total / *tgt_total */
int sqf_synthetic_corpus(int npairs, int src_vocab, int tgt_vocab, double zipf_s, uint64_t seed,
                         int32_t* src_len, int32_t* tgt_len, int32_t* src_ids, int32_t* tgt_ids,
                         int64_t* src_total, int64_t* tgt_total);
void* sqf_corpus_create(int npairs, const int32_t* src_len, const int32_t* tgt_len,
                        const int32_t* src_ids, const int32_t* tgt_ids);
void sqf_corpus_free(void* c);
/* make_batches (data.cpp:115-161) */
int sqf_make_batches(void* corpus, int64_t max_tokens, int max_sentences, uint64_t seed,
                     int32_t* nbatches, int32_t* sizes, int32_t* members);
/* shuffle_epoch (data.cpp:163-170) */
int sqf_shuffle_epoch(int nbatches, uint64_t seed, int epoch, int32_t* order);
/* make_minibatch (data.cpp:172-219): dims = {rows, src_width, tgt_width} */
int sqf_make_minibatch(void* corpus, const int32_t* members, int n, int32_t* dims, int32_t* source,
                       int32_t* target_in, int32_t* target_out, int32_t* src_lens, int32_t* tgt_lens,
                       int64_t* ntokens);
/* Trainer::split_batch (trainer.cpp:186-202): member counts per group g = w*A+a */
int sqf_split_counts(int rows, int workers, int accum, int32_t* counts);
/* bucket_gradients (trainer.cpp:50-73) */
int sqf_bucket_gradients(const int64_t* sizes, int n, int64_t threshold, int32_t* nbuckets,
                         int64_t* starts, int64_t* ends);
/* model layout + initial parameters on the host (model.cpp:74-150):
 * canonical-order params (cap >= num params) and the manifest count */
int sqf_model_init(const char* arch, const char* const* keys, const char* const* vals, int n,
                   float* params, int64_t cap, int64_t* num_params, int* manifest_size);
/* LossScaler policy (trainer.cpp:21-48) over an overflow sequence */
int sqf_scaler_run(double init, int64_t window, double mn, double mx, const uint8_t* overflow, int n,
                   double* scales, int32_t* diverged_at);
/* learning-rate schedules (optim.cpp:97-137) by registry name */
int sqf_schedule_lr(const char* name, double base, int64_t warmup, double init, double eta_min,
                    int64_t period, double t_mult, int64_t step, double* out);
/* binary16 RNE round trip (fp16.cpp:22-76) */
float sqf_quantize_fp16(float x);

/* ---- generation (reference generate.hpp:12-90, generate.cpp:123-480) ----
 * GenConfig fields; the decoder runs on the device from the trainer's compute
 * weights (fp32 master, or the fp16/bf16 shadow), incrementally with per-layer
 * K/V caches unless no_cache. */
typedef struct sqf_gen_config {
  int32_t beam;
  int32_t max_len;          /* 0 = 2 * source_len + 8 */
  int32_t diverse_groups;
  int32_t topk;
  double lenpen;
  double diverse_strength;
  double temperature;
  uint64_t seed;
  int32_t no_cache;         /* 1 = re-decode the full prefix each step (reference oracle mode) */
  int32_t host_select;      /* 1 = rank all rows x V candidates on the host instead of
                               sfk_beam_topk on the device (testing) */
} sqf_gen_config;
/* gen_config_from(trainer's resolved config) (generate.cpp:15-26) */
int sqf_gen_config_default(void* t, sqf_gen_config* out);
/* mode 0 = beam_search, 1 = diverse_beam_search, 2 = top_k_sample.
 * source: rows x src_width ids (pad 1), src_lens per row (0 = empty row);
 * stream_ids: sampling stream per row (NULL = row index). *out receives a
 * result handle (free with sqf_gen_free). */
int sqf_generate(void* t, int mode, const int32_t* source, const int32_t* src_lens, int rows, int src_width,
                 const sqf_gen_config* cfg, const uint64_t* stream_ids, void** out);
/* number of hypotheses for sentence s */
int sqf_gen_count(void* g, int s);
/* hypothesis k of sentence s: *len tokens (cap >= len, else -3), step scores */
int sqf_gen_hyp(void* g, int s, int k, int32_t* tokens, float* step_scores, int cap, int32_t* len,
                double* cum_logprob, double* score, int32_t* finish_step, int32_t* finished);
void sqf_gen_free(void* g);
/* score_hypothesis (generate.cpp:28-32) */
int sqf_score_hypothesis(double cum_logprob, int64_t length, double alpha, double* out);
/* sample_from_topk (generate.cpp:353-383) */
int sqf_sample_from_topk(const float* logits, int vocab, int k, double temperature, double u, int32_t* out);
/* batch_for_inference (generate.cpp:459-480): lens of n sources -> groups
 * (original indices, concatenated in processing order) and group sizes */
int sqf_batch_for_inference(const int32_t* lens, int n, int64_t max_tokens, int32_t* ngroups, int32_t* sizes,
                            int32_t* members);

#ifdef __cplusplus
}
#endif
#endif /* SQF_TRAINER_H */
