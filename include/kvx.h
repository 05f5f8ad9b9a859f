/*
 * kvx.h - C-ABI of the B200 (sm_100a) prefill->decode KV hand-off library.
 *
 * Reference interface being replaced
 * ----------------------------------
 * The reference (ThunderServe planner, /root/reference/pkg) ships the hand-off
 * only as an analytic model:
 *   KvPrecision            pkg/src/hetplan/costs.py:18-30   (bits in {16,8,4,2})
 *   bottleneck_link        pkg/src/hetplan/costs.py:51-65   (the P->D link)
 *   kv_comm_cost           pkg/src/hetplan/costs.py:83-103  (alpha + 2bshN_bytesL/beta)
 * called at the hand-off site pkg/src/hetplan/simulate.py:221-235 and in
 * pkg/src/hetplan/orchestrate.py:369-372.  The data path it models
 * (PAPER.md:490-493 quantise+pack -> transfer -> unpack+dequantise; NCCL
 * async SendRecv/cudaMemcpy from prefill-side KV queues) is
 * what these entry points implement.  The Python layer
 * (paper_2502_09334_b200/) keeps KvPrecision / kv_comm_cost verbatim and binds
 * these symbols with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - The caller owns every buffer; nothing here allocates on the hot path
 *    (kvx_malloc exists only for IPC-exportable staging buffers at setup).
 *  - Every compute/transfer call is stream-ordered and asynchronous; `stream`
 *    is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Return 0 on success, else a kvx/cuda error code; kvx_strerror() names it.
 *    No exceptions cross the ABI.  Re-entrant across host threads (the
 *    per-device launch caches are atomics / mutex-guarded).
 *  - Device pointers may be local, peer-mapped (kvx_enable_peer) or
 *    IPC-mapped (kvx_ipc_open): a quantise kernel writing into a peer buffer
 *    is the fused quantise+NVLink-push path, a dequantise kernel reading from
 *    a peer buffer is the fused NVLink-pull+dequantise path.
 *
 * Data layout (HBM)
 *  - KV source / destination planes are paged or dense token-major:
 *      plane(l, kv) = (kv ? v_base : k_base) + l * layer_stride    [elements]
 *      token t of a plane lives at plane + pos(t) * n_heads * head_dim
 *      pos(t) = slots ? slots[t] : t   (slots[t] < 0 = padding, skipped on
 *      the decode side; vLLM flash layout [num_blocks, block_size, H, D]
 *      has pos = block * block_size + offset).
 *  - Packed payload, per layer l (row i = (kv*n_tokens + t)*n_heads + h):
 *      codes  uint8 [2*T*H][head_dim*bits/8]  code k of a byte at bits
 *             [k*bits, (k+1)*bits) (low = even element; KIVI's int32 order)
 *      scale  fp16  [2*T*H][head_dim/group]
 *      zero   fp16  [2*T*H][head_dim/group]
 *    payload_layer_stride == 0: three dense arrays, layers back to back in
 *    each.  payload_layer_stride > 0 (bytes, multiple of 16; of 32 at 8 bits,
 *    whose codes move as 32-byte vectors): one segment per
 *    layer, codes/scale/zero of layer l at codes/scale/zero + l*stride -- a
 *    range of layers is then ONE contiguous byte range (one NVLink copy or
 *    one doorbell per layer chunk).
 *    bits == 16 is passthrough: codes are the raw fp16 rows, no scale/zero.
 *  - Arithmetic (bit-exact vs oracle/):
 *      z = f16(min + 0), s = f16((max - min)/(2^bits-1) + 0)  [IEEE fp32]
 *      q = s == 0 ? 0 : min(rint_even(RN32(x - z) * rcp_rn(s)), 2^bits-1)
 *          (the product is NOT rounded to fp32: one rounding to integer)
 *      x_hat = f16_rn(min(q*s + z, 65504))  (one rounding: fp16 FMA)
 */
#ifndef KVX_H_
#define KVX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVX_OK 0
/* kvx-specific codes live above the cudaError_t range. */
#define KVX_ERR_INVALID_ARG 10001  /* ValueError on the Python side         */
#define KVX_ERR_NO_PATH 10002      /* NoPath: no peer access between GPUs    */
#define KVX_ERR_UNSUPPORTED 10003  /* stream memory ops etc. unavailable     */
#define KVX_ERR_NCCL 10004         /* an NCCL call failed                    */

/* Library version (major*10000 + minor*100 + patch). */
int kvx_version(void);

/* Human-readable name of a return code (kvx or cudaError_t). */
const char* kvx_strerror(int code);

/* Number of CUDA devices visible (0 on a host without GPUs). */
int kvx_device_count(int* count);

/*
 * K1: per-group asymmetric quantise + pack (prefill side).
 * Replaces the 2*b*s*h*N_bytes*L "compress" term of kv_comm_cost
 * (costs.py:102) with real data.  Reads n_layers*2*n_tokens*n_heads rows of
 * head_dim fp16 from the (possibly paged: src_slots != NULL) source planes and
 * writes the dense packed payload.  codes/scale/zero may be peer pointers
 * (fused NVLink push).  bits in {2,4,8} (16 = passthrough copy, scale/zero
 * ignored); group in {32,64,128} dividing head_dim; head_dim % 8 == 0.
 * Head window (TP head shards): the source planes' token rows
 * hold plane_heads heads (0 = n_heads); only heads [head_offset,
 * head_offset + n_heads) are packed.  The payload rows then hold n_heads.
 */
int kvx_quant_pack(const void* k_src, const void* v_src, int64_t src_layer_stride,
                   const int64_t* src_slots, int64_t n_layers, int64_t n_tokens, int n_heads,
                   int head_dim, int group, int bits, void* codes, void* scale, void* zero,
                   int64_t payload_layer_stride, int plane_heads, int head_offset, void* stream);

/*
 * K1 with device-side doorbells (fused quantise -> NVLink pull pipeline):
 * same contract as kvx_quant_pack (bits 2/4/8), plus for every chunk of
 * layers_per_chunk layers the kernel itself sets peer_ready_flags[chunk] =
 * ready_value (a peer/IPC-mapped address on the decode GPU; st.release.sys)
 * as soon as the chunk's payload is complete, while it keeps quantising
 * later layers.
 * counters: 64 u32 of scratch on this GPU, zero before the first call (the
 * kernel leaves them zero again).
 * free_flag (nullable, this GPU's memory): before storing anything, every
 * CTA waits (in-kernel, bounded, abortable through ctl) until
 * *free_flag >= free_value -- the decode side's "queue slot consumed"
 * sequence number.
 * Sequence protocol (replaces round 1's parity flags): hand-off e uses
 * queue slot h = e % Q for the v-th time, v = (e - 1) / Q + 1; the prefill
 * side waits free[h] >= v - 1 and rings ready[h][c] = v, the decode side
 * waits ready[h][c] >= v and sets free[h] = v.  Values only grow, every wait
 * is the wrap-safe (int32)(flag - value) >= 0, so a doorbell left by an
 * earlier (longer) use of the slot can never satisfy a later wait.
 * ctl (nullable): a kvx_ctl_alloc'd control block; see below.
 */
int kvx_quant_pack_signal(const void* k_src, const void* v_src, int64_t src_layer_stride,
                          const int64_t* src_slots, int64_t n_layers, int64_t n_tokens,
                          int n_heads, int head_dim, int group, int bits, void* codes,
                          void* scale, void* zero, int64_t payload_layer_stride,
                          int plane_heads, int head_offset, void* counters,
                          void* peer_ready_flags, int layers_per_chunk, uint32_t ready_value,
                          const void* free_flag, uint32_t free_value, void* ctl, void* stream);

/*
 * K3: unpack + dequantise + scatter into the decode side's paged KV cache.
 * Replaces the ready = prefill_done + kv_delay step (simulate.py:235) with the
 * real decode-side enrolment.  codes/scale/zero may be peer pointers (fused
 * NVLink pull).  dst_slots[t] < 0 skips token t.  block_size is implied by the
 * slot values (pos = block*block_size + offset).  Head window as in
 * kvx_quant_pack: the cache's token rows hold plane_heads heads and this
 * payload's n_heads land at head_offset (a decode TP rank receiving part of
 * its heads from each of several prefill ranks).
 */
int kvx_dequant_scatter_paged(const void* codes, const void* scale, const void* zero,
                              int64_t payload_layer_stride, const int64_t* dst_slots,
                              int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                              int group, int bits, void* k_cache, void* v_cache,
                              int64_t dst_layer_stride, int plane_heads, int head_offset,
                              void* stream);

/*
 * K3 with TMA bulk staging: same contract as kvx_dequant_scatter_paged, but
 * the payload is streamed into shared memory with cp.async.bulk (one request
 * per span of token rows) -- the fused NVLink-pull variant for a payload that
 * lives in the prefill GPU's HBM.
 * ready_flags (nullable, this GPU's memory): the kernel itself waits, per
 * chunk of layers_per_chunk layers, until ready_flags[chunk] >= ready_value,
 * so ONE launch consumes a whole hand-off while the prefill GPU is still
 * producing it (kvx_quant_pack_signal, or kvx_stream_signal after each
 * chunk's K1).  Without flags, shapes whose rows are not 16-byte multiples
 * fall back to the per-lane kernel; with flags they return
 * KVX_ERR_UNSUPPORTED (see kvx_pull_supported).
 * done_counter / peer_free_flag (nullable, together): in-kernel completion --
 * done_counter is a u32 on this GPU (0 before the first call, left 0); the
 * last CTA sets *peer_free_flag = ready_value (a peer/IPC-mapped u32 on the
 * prefill GPU: "queue slot consumed") unless the wait was aborted.
 * flags: KVX_PULL_PDL launches with programmatic stream serialization -- the
 * kernel's producer may start pulling this hand-off's slot while the
 * stream's previous kernel (typically the previous hand-off's pull) is still
 * running; everything that touches stream-ordered memory (the slot mapping,
 * the cache, done_counter) waits for it (griddepcontrol.wait).
 * KVX_PULL_CHAINED (with KVX_PULL_PDL): the caller promises that the stream's
 * previous kernel is a pull of the same pair, and -- for the whole run of
 * chained pulls since the last unchained one -- that every slot mapping was
 * ready before the run started and that no two pulls of the run write the
 * same cache blocks (several of them may be writing at once).  The
 * consumers then write while the previous pulls drain; only the completion
 * (done_counter, the free flag) waits, so pulls complete in order and an
 * unchained pull after the run starts after all of them.
 */
#define KVX_PULL_PDL 1
#define KVX_PULL_CHAINED 2
int kvx_pull_dequant_scatter_paged(const void* codes, const void* scale, const void* zero,
                                   int64_t payload_layer_stride, const int64_t* dst_slots,
                                   int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                                   int group, int bits, void* k_cache, void* v_cache,
                                   int64_t dst_layer_stride, int plane_heads, int head_offset,
                                   const void* ready_flags, uint32_t ready_value,
                                   int layers_per_chunk, void* done_counter, void* peer_free_flag,
                                   void* ctl, int flags, void* stream);

/* 1 if kvx_pull_dequant_scatter_paged can bulk-stage this shape. */
int kvx_pull_supported(int64_t n_tokens, int n_heads, int head_dim, int group, int bits);

/*
 * "kivi" format (KIVI-style): K quantised PER CHANNEL over
 * groups of `group` (32|64) consecutive tokens of one request -- the group
 * starts are group_starts[n_groups] in batch token order -- and each request's
 * last n % group tokens (residual_tokens[n_residual]) sent as fp16; V per
 * token (group along head_dim) as in the default format.  bits in {4, 8};
 * dense sources only.  Payload: one segment per layer (payload_layer_stride
 * bytes) holding seven 16-B aligned sub-arrays at seg_offsets[7] (host array):
 *   Kc u8 [n_groups*group][H][D*bits/8] (group-major rows)
 *   Ks, Kz f16 [n_groups][H][D]   Kr f16 [n_residual][H][D]
 *   Vc u8 [T][H][D*bits/8]        Vs, Vz f16 [T][H][D/group]
 * Decode side: dst_slots[T] for every token, residual_dst_slots[n_residual]
 * = dst_slots[residual_tokens].
 */
int kvx_quant_pack_kivi(const void* k_src, const void* v_src, int64_t src_layer_stride,
                        int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim, int group,
                        int bits, const int64_t* group_starts, int64_t n_groups,
                        const int64_t* residual_tokens, int64_t n_residual, void* payload,
                        int64_t payload_layer_stride, const int64_t* seg_offsets, void* stream);
int kvx_dequant_scatter_paged_kivi(const void* payload, int64_t payload_layer_stride,
                                   const int64_t* seg_offsets, const int64_t* dst_slots,
                                   const int64_t* group_starts, int64_t n_groups,
                                   const int64_t* residual_dst_slots, int64_t n_residual,
                                   int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                                   int group, int bits, void* k_cache, void* v_cache,
                                   int64_t dst_layer_stride, void* stream);
/*
 * Fused kivi prefill side: kvx_quant_pack_kivi over a whole hand-off with
 * device doorbells (no per-chunk launches or stream memops).  The K
 * (per-channel) quantiser sets peer_ready_flags[c] = ready_value as soon as
 * chunk c (layers_per_chunk layers; at most KVX_KIVI_V_FLAGS chunks) of K
 * is in the payload; the residual rows follow; the V quantiser then sets
 * peer_ready_flags[KVX_KIVI_V_FLAGS + c] per chunk -- a V doorbell publishes
 * the whole chunk (K, residual and V).  peer_ready_flags may be IPC/peer
 * mapped (st.release.sys).  counters: 2*64 u32 of scratch on this GPU, zero
 * before the first call (left zero).  free_flag (nullable): the launches are
 * held in the GPU front-end (stream memop) until *free_flag >= free_value
 * (the queue slot's previous use consumed).  ctl as for kvx_quant_pack_signal.
 */
#define KVX_KIVI_V_FLAGS 32
int kvx_quant_pack_kivi_signal(const void* k_src, const void* v_src, int64_t src_layer_stride,
                               int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                               int group, int bits, const int64_t* group_starts, int64_t n_groups,
                               const int64_t* residual_tokens, int64_t n_residual, void* payload,
                               int64_t payload_layer_stride, const int64_t* seg_offsets,
                               void* counters, void* peer_ready_flags, int layers_per_chunk,
                               uint32_t ready_value, const void* free_flag, uint32_t free_value,
                               void* ctl, void* stream);
/* Same contract as kvx_dequant_scatter_paged_kivi, for a payload read over
 * NVLink: the per-channel K groups and
 * the per-token V rows are staged into shared memory with cp.async.bulk
 * (TMA) before they are dequantised -- the kivi format's pull transport.
 * Shapes that cannot be bulk-staged fall back to the per-lane kernels.
 * ready_flags (nullable, this GPU's memory): the kernels wait in-kernel, per
 * chunk of layers_per_chunk layers, until the chunk's doorbell is >=
 * ready_value -- K groups on ready_flags[chunk], V rows (and, after them,
 * the residual rows) on ready_flags[KVX_KIVI_V_FLAGS + chunk], the layout
 * kvx_quant_pack_kivi_signal rings -- so ONE call consumes a whole hand-off
 * while the prefill side is still publishing it.  done_counter /
 * peer_free_flag (nullable, together; only with ready_flags): the queue slot
 * is released once the hand-off's last payload read is done -- by the single
 * kivi pull kernel's last CTA, or in stream order after the residual rows on
 * the two-kernel fallback; without them the caller releases it.  flags: KVX_PULL_PDL launches both pulls
 * with programmatic dependent launch (each one's producer streams while the
 * stream's previous kernel drains).  With flags, shapes that cannot be bulk-staged return
 * KVX_ERR_UNSUPPORTED.  ctl as for kvx_quant_pack_signal.
 * 8-bit: seg_offsets[4] (V codes) and payload_layer_stride must be 32-byte
 * multiples (32-byte vector accesses). */
int kvx_pull_dequant_scatter_paged_kivi(const void* payload, int64_t payload_layer_stride,
                                        const int64_t* seg_offsets, const int64_t* dst_slots,
                                        const int64_t* group_starts, int64_t n_groups,
                                        const int64_t* residual_dst_slots, int64_t n_residual,
                                        int64_t n_layers, int64_t n_tokens, int n_heads,
                                        int head_dim, int group, int bits, void* k_cache,
                                        void* v_cache, int64_t dst_layer_stride,
                                        const void* ready_flags, uint32_t ready_value,
                                        int layers_per_chunk, void* done_counter,
                                        void* peer_free_flag, void* ctl, int flags,
                                        void* stream);

/* Packed payload sizes in bytes for n_rows rows (codes, scale, zero). */
int kvx_packed_sizes(int64_t n_rows, int head_dim, int group, int bits, int64_t* codes_bytes,
                     int64_t* scale_bytes, int64_t* zero_bytes);

/* ---- transport: NVLink P2P within one process --------------------------- */

/* Enable peer access a->b and b->a (idempotent).  KVX_ERR_NO_PATH if the
 * devices cannot access each other (costs.py:63-64 raises NoPath there). */
int kvx_enable_peer(int dev_a, int dev_b);

/* Copy-engine peer copy (cudaMemcpyPeerAsync): the non-fused baseline. */
int kvx_copy_peer(void* dst, int dst_dev, const void* src, int src_dev, size_t n_bytes,
                  void* stream);

/* ---- transport: NVLink P2P across processes (one process per GPU) ------- */

/* cudaMemcpyAsync with cudaMemcpyDefault (unified addressing): any mix of
 * host-pinned, local, peer and IPC-mapped addresses (doorbell polling,
 * staging). */
int kvx_memcpy_async(void* dst, const void* src, size_t n_bytes, void* stream);

/* IPC-exportable device allocation (setup only, never on the hot path). */
int kvx_malloc(void** ptr, size_t n_bytes);
int kvx_free(void* ptr);
int kvx_memset_async(void* ptr, int value, size_t n_bytes, void* stream);

/* cudaIpcMemHandle_t export / import (64 opaque bytes). ptr must be a
 * kvx_malloc base pointer.  kvx_ipc_open maps a peer's buffer into this
 * process (peer access implied); kvx_ipc_close unmaps it. */
int kvx_ipc_handle_size(void);
int kvx_ipc_get_handle(void* ptr, void* handle_out);
int kvx_ipc_open(const void* handle, void** ptr_out);
int kvx_ipc_close(void* ptr);

/* Stream-ordered 32-bit flags (cuStreamWriteValue32 / cuStreamWaitValue32)
 * used as cross-GPU chunk doorbells: the producer signals after the chunk's
 * kernel (with a memory barrier), the consumer's stream blocks in the
 * front-end (no spinning kernel) until flag >= value (wrap-safe), or, for
 * kvx_stream_wait_eq, until flag == value.  flag may be a local, peer or
 * IPC-mapped device address. */
int kvx_stream_signal(void* flag, uint32_t value, void* stream);
int kvx_stream_wait(const void* flag, uint32_t value, void* stream);
int kvx_stream_wait_eq(const void* flag, uint32_t value, void* stream);
/* 1 if stream memory operations are usable on the current device. */
int kvx_stream_memops_supported(int* supported);

/* ---- control block: abort and timeout of the in-kernel waits ------------- */

/* A channel's control block, in host memory mapped into every GPU (UVA: the
 * kernels use the host address).  The host sets `abort` to make every
 * kernel spinning on one of the channel's doorbells wind down; a kernel whose
 * wait is aborted or outlives `timeout_ns` (0 = 60 s) records
 * KVX_STATUS_ABORTED / KVX_STATUS_TIMEOUT in `status` and exits cleanly
 * instead of trapping -- the CUDA context and the decode GPU's cache survive
 * a lost partner; the Python layer raises PartnerLost (a NoPath). */
typedef struct kvx_ctl {
  uint32_t abort;      /* host -> device: nonzero = give up waiting      */
  uint32_t status;     /* device -> host: 0 ok, KVX_STATUS_*              */
  uint64_t timeout_ns; /* bound of every in-kernel wait (0 = 60 s)        */
} kvx_ctl;
#define KVX_STATUS_OK 0
#define KVX_STATUS_ABORTED 1
#define KVX_STATUS_TIMEOUT 2
int kvx_ctl_alloc(void** ctl_out); /* zeroed, cudaHostAlloc(Mapped|Portable) */
int kvx_ctl_free(void* ctl);

/* ---- the pair channel: one end of a prefill -> decode pair ---------------- */

/* Layer chunks of one pull hand-off of n_tokens tokens (identical on both
 * ends): layer-granular doorbells (<= 64 chunks) with at least 4 K1 items per
 * resident K1 warp in each, or every layer its own chunk (<= 64) when
 * `layerwise` (streaming during prefill). */
int kvx_handoff_chunk_plan(int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                           int layerwise, int* layers_per_chunk, int* n_chunks);

/* One end of a prefill -> decode pair over the sequence protocol above,
 * mirroring the paper's pre-built P2P group pool with KV queues in prefill
 * GPU memory.  The caller maps the memory (CUDA IPC or peer
 * access) and owns it:
 *   local_flags / peer_flags: this GPU's and the partner's 4 KB doorbell
 *     pages (u32 ready[8][64] at 0, free[8] at 512);
 *   payload: the prefill GPU's queue, queue_depth slots of slot_bytes
 *     (256-B aligned, each >= n_layers * the 256-B aligned per-layer segment
 *     of max_tokens tokens); local on the prefill end, mapped on the decode
 *     end;  ctl: nullable control block.
 * The pair allocates Q x 65 u32 of device scratch at creation; send/recv
 * never allocate.  Hand-off e (1, 2, ... in the same order on both ends) is
 * ONE kernel launch per end:
 *   kvx_pair_send: K1 with device doorbells into slot e % Q (KVX_PAIR_GATE:
 *     first a stream memop holding the launch in the GPU front-end until the
 *     decode side has freed the slot -- a lagging partner holds no SMs;
 *     KVX_PAIR_PDL instead: latency mode, the K1 is launched with
 *     programmatic dependent launch behind the stream's previous kernel and
 *     waits for the slot in-kernel only);
 *   kvx_pair_recv: K3-bulk pulling the slot over NVLink as chunks are
 *     published, freeing it in-kernel (KVX_PAIR_GATE: launch once chunk 0 is
 *     published; KVX_PAIR_PDL: programmatic dependent launch, so a pull
 *     streams its slot while the previous hand-off's pull drains;
 *     KVX_PAIR_CHAINED with KVX_PAIR_PDL: KVX_PULL_CHAINED's promise --
 *     a run of back-to-back recvs, each into blocks no other recv of the run
 *     writes, slot mappings ready before the run -- so the pull also writes
 *     the cache while earlier pulls drain).
 * Validation: n_tokens <= max_tokens, the head window inside the planes, the
 * current device == the creating device.  Replaces the kv_delay the
 * reference charges per request (simulate.py:221-235). */
#define KVX_ROLE_PREFILL 0
#define KVX_ROLE_DECODE 1
#define KVX_PAIR_GATE 1
#define KVX_PAIR_PDL 2
#define KVX_PAIR_CHAINED 4
int kvx_pair_create(int role, int64_t n_layers, int64_t max_tokens, int n_heads, int head_dim,
                    int bits, int group, int queue_depth, int layerwise, void* local_flags,
                    void* peer_flags, void* payload, int64_t slot_bytes, void* ctl,
                    void** pair_out);
int kvx_pair_send(void* pair, uint64_t epoch, const void* k_src, const void* v_src,
                  int64_t src_layer_stride, const int64_t* src_slots, int64_t n_tokens,
                  int plane_heads, int head_offset, int flags, void* stream);
int kvx_pair_recv(void* pair, uint64_t epoch, void* k_cache, void* v_cache,
                  int64_t dst_layer_stride, const int64_t* dst_slots, int64_t n_tokens,
                  int plane_heads, int head_offset, int flags, void* stream);
/* Decode end: ONE K3-bulk launch pulling `count` consecutive hand-offs
 * (epochs first_epoch .. first_epoch + count - 1, count <= queue_depth, <= 8)
 * into the same paged cache -- the decode side draining everything queued
 * after a decode round.  dst_slots / n_tokens: HOST arrays of
 * `count` device slot-mapping pointers and token counts (each >= 1).  Each
 * part waits on its own chunk doorbells in-kernel; the last CTA frees every
 * part's queue slot.  flags: KVX_PAIR_PDL only.  KVX_ERR_UNSUPPORTED for a
 * shape the bulk pull cannot stage (use kvx_pair_recv per hand-off). */
int kvx_pair_recv_many(void* pair, uint64_t first_epoch, int count, void* k_cache, void* v_cache,
                       int64_t dst_layer_stride, const int64_t* const* dst_slots,
                       const int64_t* n_tokens, int plane_heads, int head_offset, int flags,
                       void* stream);
int kvx_pair_destroy(void* pair);

/* ---- NCCL pair pool ---------------------------
 * The paper pre-builds NCCL groups for its asynchronous SendRecv hand-offs;
 * these mirror that for engines that pair GPUs through NCCL (TP-sharded
 * replicas, or pairings without CUDA IPC).  NCCL is resolved at run time
 * (the process's already-loaded libnccl.so.2, else the system one):
 * KVX_ERR_UNSUPPORTED without it, KVX_ERR_NCCL when a call fails.
 *   kvx_nccl_get_unique_id: 128 opaque bytes (rank 0; the caller broadcasts)
 *   kvx_nccl_pair_init: ncclCommInitRank (collective over the n_ranks)
 *   kvx_nccl_sendrecv: ONE ncclGroupStart/End holding a send of send_bytes to
 *     send_peer and a receive of recv_bytes from recv_peer (a peer < 0 or 0
 *     bytes skips that half), stream-ordered on `stream` -- e.g. a packed
 *     payload (kvx_quant_pack) on the prefill rank, the landing buffer of
 *     kvx_dequant_scatter_paged on the decode rank. */
int kvx_nccl_unique_id_size(void);
int kvx_nccl_get_unique_id(void* id_out);
int kvx_nccl_pair_init(const void* unique_id, int n_ranks, int rank, void** comm_out);
int kvx_nccl_sendrecv(void* comm, const void* send_buf, size_t send_bytes, int send_peer,
                      void* recv_buf, size_t recv_bytes, int recv_peer, void* stream);
int kvx_nccl_pair_destroy(void* comm);

#ifdef __cplusplus
}
#endif

#endif /* KVX_H_ */
