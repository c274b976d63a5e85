/*
 * hegpu.h -- C-ABI of the B200-native CKKS/RNS backend (libhegpu.so).
 *
 * This is the drop-in boundary for the reference's HE backend hot path
 * (arxiv/paper_1810_10121 "hegraph"; paths below are relative to
 * /root/reference/proj/include/heg/).  Host C++ (graph, planning, keys,
 * encoders) calls sm_100a CUDA through these entry points; no C++ or torch
 * types cross it: plain pointers, sizes and status codes.
 *
 * Conventions
 *  - Every function returns 0 on success or an HG_E* code (mirrors heg::errc,
 *    common.hpp:37-46, plus HG_ECUDA) and never throws; hg_last_error()
 *    returns the message of the last failure on the calling thread.  The
 *    messages match the reference's heg::Error texts where one exists.
 *  - Ciphertext buffers are DEVICE pointers to uint64 words laid out
 *    [item][poly][limb][N] (the reference's RnsPoly residue order,
 *    poly.hpp:35-41), NTT form unless stated, `nl` = level + 1 limbs.
 *  - Work is issued on the context's stream (hg_context_stream); functions
 *    returning host data synchronise that stream.
 */
#ifndef HEGPU_H
#define HEGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_OK 0
#define HG_E_VALIDATION 1 /* errc::validation */
#define HG_E_PARSE 2      /* errc::parse */
#define HG_E_DEPTH 3      /* errc::depth_exceeded */
#define HG_E_CAPACITY 4   /* errc::capacity */
#define HG_E_IO 5         /* errc::io */
#define HG_E_INTERNAL 6   /* errc::internal */
#define HG_E_CUDA 7       /* CUDA runtime failure */

typedef struct hg_context hg_context;
typedef struct hg_keys hg_keys;
typedef struct hg_plan hg_plan;
typedef struct hg_output hg_output;

const char* hg_last_error(void);
const char* hg_version(void);

/* ---- context (replaces heg::make_context / CryptoContext, context.hpp:90-165) ---- */
int hg_context_create(int64_t poly_degree, const int* coeff_mod_bits, int nbits, int scale_bits, int security,
                      int device, hg_context** out);
void hg_context_destroy(hg_context* ctx);
/* the ContextParams a context was built from (ring degree, coeff_mod_bits, scale_bits, security) */
int hg_context_params(const hg_context* ctx, int64_t* n, int* bits, int cap, int* nbits, int* scale_bits,
                      int* security);
/* writes up to `cap` primes; returns the prime count via *count */
int hg_context_primes(const hg_context* ctx, uint64_t* primes, int cap, int* count);
/* relin digit counts D_i (ckks_backend.hpp:42-46) and total rows */
int hg_context_relin_rows(const hg_context* ctx, int* rows);
/* issue work on an external cudaStream_t (e.g. torch's current stream; NULL = legacy default stream) */
int hg_context_set_stream(hg_context* ctx, void* cuda_stream);
/* back to the context's private non-blocking stream */
int hg_context_use_private_stream(hg_context* ctx);
void* hg_context_stream(const hg_context* ctx);
int hg_sync(const hg_context* ctx);

/* ---- keys (replaces heg::ckks::generate_keys, ckks_backend.hpp:74-114) ---- */
int hg_keys_generate(hg_context* ctx, uint64_t seed, int with_relin, hg_keys** out);
void hg_keys_destroy(hg_keys* keys);
/* host copies, NTT form, full chain: secret[(L+1)N], pk[2][(L+1)N], relin[rows][2][(L+1)N] (relin may be NULL) */
int hg_keys_export(const hg_context* ctx, const hg_keys* keys, uint64_t* secret, uint64_t* pk, uint64_t* relin);

/* ---- key and ciphertext files (keyio.hpp:36-302: HEGK / HEGC, coefficient-domain u64 LE) ----
 * Byte-identical to the reference's save_keys / save_ciphertext; loading re-homes the
 * payload into the GPU's NTT-form residency. */
int hg_keys_save(const hg_context* ctx, const hg_keys* keys, const char* path);
/* load_keys (keyio.hpp:171-238): builds the context from the file's header on `device` */
int hg_keys_load(const char* path, int device, hg_context** ctx_out, hg_keys** keys_out);
/* save_ciphertext (keyio.hpp:244-259) of a device ciphertext [size][level+1][N] (NTT form) */
int hg_ciphertext_save(hg_context* ctx, const uint64_t* ct_dev, int size, int level, double scale, const char* path);
/* load_ciphertext (keyio.hpp:267-293); ct_dev NULL = header only (size, level, scale) */
int hg_ciphertext_load(hg_context* ctx, const char* path, uint64_t* ct_dev, int64_t capacity_words, int* size,
                       int* level, double* scale);

/* ---- ring kernels (NttTables::forward/inverse, ring.hpp:263-301) ---- */
/* in-place on `rows` limb rows; row r is limb (r % nl) at dev + r*N */
int hg_ntt_forward(hg_context* ctx, uint64_t* dev, int64_t rows, int nl);
int hg_ntt_inverse(hg_context* ctx, uint64_t* dev, int64_t rows, int nl);

/* ---- ciphertext primitives (CkksBackend, ckks_backend.hpp:253-377) ---- */
int hg_add(hg_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t words, int nl);
int hg_sub(hg_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t words, int nl);
int hg_negate(hg_context* ctx, const uint64_t* a, uint64_t* out, int64_t words, int nl);
/* poly 0 of each item +/- plaintext (pt_per_item: pt has one [nl][N] block per item, else shared) */
int hg_add_plain(hg_context* ctx, const uint64_t* ct, const uint64_t* pt, uint64_t* out, int64_t items, int size,
                 int nl, int pt_per_item, int subtract);
int hg_multiply_plain(hg_context* ctx, const uint64_t* ct, const uint64_t* pt, uint64_t* out, int64_t items, int size,
                      int nl, int pt_per_item);
/* rescale `polys` polys from nl to nl-1 limbs (poly_rescale, poly.hpp:190-228) */
int hg_rescale(hg_context* ctx, const uint64_t* in, uint64_t* out, int64_t polys, int nl);
int hg_mod_switch(hg_context* ctx, const uint64_t* in, uint64_t* out, int64_t polys, int nl_in, int nl_out);
/* size-2 x size-2 -> relinearised size-2 (multiply + relinearize, ckks_backend.hpp:261-281, 508-554) */
int hg_multiply_relin(hg_context* ctx, const hg_keys* keys, const uint64_t* a, const uint64_t* b, uint64_t* out,
                      int64_t items, int nl);
/* size-2 x size-2 -> size-3 tensor only */
int hg_multiply_tensor(hg_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out3, int64_t items, int nl);
int hg_relinearize(hg_context* ctx, const hg_keys* keys, const uint64_t* in3, uint64_t* out2, int64_t items, int nl);
/* fused multiply+relin+rescale of x by itself (PolyAct x^2 -> multiply_rescale(x, x)) -> nl-1 limbs */
int hg_square_relin_rescale(hg_context* ctx, const hg_keys* keys, const uint64_t* in, uint64_t* out, int64_t items,
                            int nl);
/* Grouped weighted sum + single rescale (weighted_sum, ckks_backend.hpp:381-411; the Dot/Convolution
 * contraction, runtime.hpp:1027-1221).  x: size-2 items at nl limbs; groups share an input list:
 *   out[g*mg+m] = rescale( sum_t  W[(g*mg+m)*kt + t][limb] * x[idx[g*kt+t]] )
 * w: device residues [(groups*mg)*kt][nl]; idx: device int32 [groups*kt]. out has nl-1 limbs. */
int hg_weighted_sum(hg_context* ctx, const uint64_t* x, const int32_t* idx, const uint64_t* w, uint64_t* out,
                    int64_t groups, int mg, int kt, int nl);
/* Ciphertext-weight sum (weighted_sum_cipher, ckks_backend.hpp:413-450; the EncryptedBoth /
 * EncryptedModel contraction, runtime.hpp:1053-1073, 605-617):
 *   out[g] = rescale( relinearize( sum_t  x[xidx[g*kt+t]] (x) w[widx[g*kt+t]] ) )
 * x, w: size-2 items at nl limbs, same level and scales; xidx, widx: device int32 [groups*kt].
 * The size-3 products are accumulated exactly, relinearised ONCE and rescaled once. */
int hg_weighted_sum_cipher(hg_context* ctx, const hg_keys* keys, const uint64_t* x, const int32_t* xidx,
                           const uint64_t* w, const int32_t* widx, uint64_t* out, int64_t groups, int kt, int nl);

/* ---- encoding / encryption (ckks_backend.hpp:182-249) ---- */
/* values (host or device) -> device plaintext (NTT form, nl = level+1 limbs).  Replaces
 * CkksBackend::encode (ckks_backend.hpp:182-197); the fp64 FFT + llround run on the GPU,
 * bit-identical to the reference's SlotEncoder (encoder.hpp:58-77). */
int hg_encode(hg_context* ctx, const double* values, int64_t count, int level, double scale, uint64_t* pt_dev);
/* `cols` plaintexts at once: slot m of column e is values[e*col_stride + m*elem_stride]
 * (pack_cipher's batch columns, packing.hpp:57-63, read straight from a [batch][elements]
 * array with col_stride = 1, elem_stride = elements).  pt_dev: [cols][level+1][N]. */
int hg_encode_batch(hg_context* ctx, const double* values, int64_t cols, int64_t count, int64_t col_stride,
                    int64_t elem_stride, int level, double scale, uint64_t* pt_dev);
/* scalar -> per-limb residues of llround(value*scale) (host array of level+1 words) */
int hg_encode_constant(hg_context* ctx, double value, int level, double scale, uint64_t* residues_host);
/* write those residues into every slot of a device plaintext (the NTT form of a constant) */
int hg_fill_constant(hg_context* ctx, const uint64_t* residues_host, int level, uint64_t* pt_dev);
/* decode a device plaintext (NTT form) to `count` slot values (CkksBackend::decode) */
int hg_decode(hg_context* ctx, const uint64_t* pt_dev, int level, double scale, int64_t count, double* values_host);
/* items fresh encryptions at `level`, seeds[item] (host), optional plaintexts pt_dev[item][nl][N] */
int hg_encrypt(hg_context* ctx, const hg_keys* keys, const uint64_t* pt_dev, const uint64_t* seeds, int64_t items,
               int level, uint64_t* out);
/* fresh-encryption samples (u, e0, e1; poly.hpp:257-276 streams of ckks_backend.hpp:470-490) as signed
 * int64 [items][3][N]: on the GPU (device out) or with the host sampler (host out) */
int hg_sample_encryption(hg_context* ctx, const uint64_t* seeds, int64_t items, int64_t* out_dev);
int hg_sample_encryption_host(hg_context* ctx, const uint64_t* seeds, int64_t items, int64_t* out_host);
/* coefficient-domain m = c0 + c1 s (+ ...) -> host [items][nl][N] */
int hg_decrypt_coeffs(hg_context* ctx, const hg_keys* keys, const uint64_t* ct, int64_t items, int size, int level,
                      uint64_t* m_host);
/* CRT reconstruction and slot decode of decrypted outputs (ring.hpp:438-480, encoder.hpp:80-89)
 * on the GPU (1, default) or on the host (0); the values are bit-identical either way */
int hg_set_gpu_decode(int on);
/* decrypt + CRT + decode to `count` slot values per item (host [items][count]) */
int hg_decrypt(hg_context* ctx, const hg_keys* keys, const uint64_t* ct, int64_t items, int size, int level,
               double scale, int64_t count, double* values_host);

/* ---- graph execution (heg::execute, runtime.hpp:1970-1974) ---- */
/* Load a format_version-1 graph (graph_io.hpp) and plan it for `batch` slots. */
int hg_plan_create(hg_context* ctx, const hg_keys* keys, const char* graph_json, int64_t batch, uint64_t exec_seed,
                   hg_plan** out);
void hg_plan_destroy(hg_plan* plan);
/* encode + encrypt a Parameter's batch (host row-major values, batch * prod(shape[1:]))  */
/* ExecOptions (runtime.hpp:158-166) as JSON, before binding inputs: {"paradigm": "encrypted-data" |
 * "encrypted-model" | "encrypted-both", "bypass": {"optimized_multiply": bool,
 * "optimized_addition": bool, "epsilon": double}}.  Replaces the ExecOptions argument of
 * heg::execute (runtime.hpp:1970-1974); the default is encrypted-data with bypass on, eps 0. */
int hg_plan_set_options(hg_plan* plan, const char* options_json);
int hg_plan_bind_input(hg_plan* plan, const char* param_id, const double* values, int64_t count);
/* server-side graph run: ciphertexts stay in HBM, no host round trip between nodes */
int hg_plan_run(hg_plan* plan);
/* decrypt + decode an output tensor (host row-major batch * elements) */
int hg_plan_output(hg_plan* plan, const char* output_id, double* values, int64_t capacity, int64_t* count);
/* raw output ciphertext access: element count, level, scale; NTT-form words copied to host or device */
int hg_plan_output_info(hg_plan* plan, const char* output_id, int64_t* elements, int* level, double* scale);
int hg_plan_output_ciphertexts(hg_plan* plan, const char* output_id, uint64_t* dst, int dst_is_device);
/* replace a Parameter's bound ciphertexts from host/device NTT-form words (client-encrypted inputs) */
int hg_plan_input_info(hg_plan* plan, const char* param_id, int64_t* elements, int* level);
int hg_plan_set_input_ciphertexts(hg_plan* plan, const char* param_id, const uint64_t* src, int src_is_device);
/* Pipelined output: enqueue the GPU decrypt + device->host copy of an output now and
 * decode it on a host thread (overlapping the next step's GPU work); the ticket is
 * consumed by hg_output_wait, which returns the same values as hg_plan_output.  The
 * output tensor may be replaced by the next hg_plan_run once this call returns. */
int hg_plan_output_async(hg_plan* plan, const char* output_id, hg_output** ticket);
int hg_output_count(const hg_output* ticket, int64_t* count);
int hg_output_wait(hg_output* ticket, double* values, int64_t capacity, int64_t* count);
/* ExecProfile (runtime.hpp:140-156) as JSON */
int hg_plan_profile_json(hg_plan* plan, char* buf, size_t cap);
/* kernel launches issued by the last hg_plan_run */
int64_t hg_plan_launches(const hg_plan* plan);

/* ---- output-sharded multi-GPU execution (one process per GPU, NCCL over NVLink) ----
 * The reference runs each layer's outputs as independent parallel_for bodies
 * (common.hpp:134-140, runtime.hpp:1104-1221); here every Dot/Conv computes only
 * this rank's block of outputs (conv windows / Dot rows, else Dot columns), x^2
 * runs on the shard, and a tensor is all-gathered (grouped in-place NCCL
 * broadcasts) where a consumer needs every element.  Results are bit-identical
 * to the unsharded run on every rank. */
/* 128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it, e.g. via torch.distributed) */
int hg_comm_unique_id(void* id_out);
/* one-rank self-test of the NCCL transport on the context's GPU: loads libnccl, creates a 1-rank
 * communicator and runs the transport's all-gather-v (grouped in-place broadcasts) over `ranges`
 * item ranges of `item_words` words; 0 on success */
int hg_comm_selftest(hg_context* ctx, int ranges, int64_t item_words);
/* join a `world`-rank group as `rank` on the plan's device; world == 1 turns sharding off */
int hg_plan_set_comm(hg_plan* plan, int rank, int world, const void* id);
/* host-mediated transport instead of NCCL (tests, or a deployment with its own collective): at
 * every gather point the plan's stream is synchronised and fn is called with the tensor's device
 * buffer `dev` (items of item_words uint64 words); ranges holds, rank by rank, counts[r] pairs of
 * [begin, end) item ranges that rank r computed; fn must fill every other rank's ranges and
 * return 0.  Same partition and gather schedule as hg_plan_set_comm. */
typedef int (*hg_gather_fn)(void* user, const char* tensor_id, uint64_t* dev, int64_t item_words,
                            const int64_t* ranges, const int32_t* counts, int world);
int hg_plan_set_gather_callback(hg_plan* plan, int rank, int world, hg_gather_fn fn, void* user);
/* in-process group on ONE device (checks the sharded path without NCCL): the plans, which
 * share one context, run in lockstep, each computing its shard; gathers are device copies */
int hg_group_run(hg_plan** plans, int world);
/* the partition rule (host only): rank's block [g0,g1) x [m0,m1) of a contraction with
 * `groups` input windows x `mg` outputs per window -> out4 = {g0, g1, m0, m1} */
int hg_shard_partition(int64_t groups, int64_t mg, int world, int rank, int64_t* out4);

/* ---- measurement hooks (bench.py) ---- */
/* record CUDA events around every kernel launch of this context (off by default) */
int hg_kernel_timing(hg_context* ctx, int on);
/* {"kernel": {"launches": n, "total_ms": t}, ...} for the launches recorded since the last call */
int hg_kernel_stats_json(hg_context* ctx, char* buf, size_t cap);
/* kernel launches issued by this context so far (counted at every launch site) */
int64_t hg_kernel_launches(const hg_context* ctx);
/* register-only modmul throughput on all SMs: wide 0 = 32-bit Shoup, 1 = 64-bit Shoup, 2 = fp64 (q < 2^50) */
int hg_bench_modmul(hg_context* ctx, int wide, double* modmul_per_s);

#ifdef __cplusplus
}
#endif
#endif
