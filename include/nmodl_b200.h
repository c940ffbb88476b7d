/* nmodl_b200.h -- C-ABI of the B200 nrn_state/nrn_cur backend.
 *
 * Two shared objects sit behind this boundary; both take plain pointers and
 * sizes only (no PyTorch or Python types):
 *
 *  1. libnmodl_b200_rt.so  (paper_1905_02241_b200/csrc/nmodl_rt.cu)
 *     device memory, streams, events, graph capture, status block,
 *     finiteness scan, checksums, node_index scatter layout.
 *  2. lib<mech>-<hash>.so  (generated per mechanism by emit_cuda,
 *     paper_1905_02241_b200/codegen_cuda.py) exporting the kernel entry
 *     points declared by NMODL_B200_MECHANISM(mech) below, over a
 *     mechanism-specific `<mech>_data` struct; see include/mechanisms/<mech>.h
 *     for the generated struct of each benchmarked mechanism.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/modlc):
 *   - emitted kernels `void <mech>_{initialize,state_update,current_update}
 *     (<mech>_data *md)`                                   codegen.py:56-61,450-455
 *   - emitted instance struct `<mech>_data`                codegen.py:425-437
 *   - `modlc_lu_solve(a, b, x, k)`                         codegen.py:540-565
 *     (now straight-line register code emitted per solve by the printer)
 *   - `Runner.run_kernel(data, kernel_name, steps)`        interp.py:456-471
 *     (the Python CudaRunner calls the entry points below through ctypes)
 *   - `InterpError` conditions                             interp.py:285,406,538,619
 *     (reported through nmodl_status)
 *
 * All functions return 0 on success or a cudaError_t code; the message of the
 * last failure is nmodl_last_error().
 */
#ifndef NMODL_B200_H
#define NMODL_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *nmodl_stream_t;  /* cudaStream_t */
typedef void *nmodl_event_t;   /* cudaEvent_t */
typedef void *nmodl_graph_t;   /* cudaGraphExec_t */

#ifndef NMODL_B200_STATUS_H
#define NMODL_B200_STATUS_H
#define NMODL_NO_ERROR 0xffffffffffffffffull
/* Device status block.  err_key is the minimum lexicographic error key
 * (kernel, phase, ordinal, kind, sub, instance) proposed by any failing lane;
 * see csrc/include/nmodl_b200/mechanism.cuh nmodl::err_key.  Replaces the
 * reference C's `long solver_failures` counter (codegen.py:239) and carries
 * what the reference runtime raises as InterpError (interp.py:285,406,538,619). */
typedef struct nmodl_status {
  unsigned long long err_key;
  unsigned long long payload_key;
  double payload;
  int lock;
  int reserved;
} nmodl_status;
#define NMODL_KIND_WHILE 0
#define NMODL_KIND_NEWTON 1
#define NMODL_KIND_SINGULAR 2
#endif

/* ---- runtime library (libnmodl_b200_rt.so) ---------------------------- */
const char *nmodl_last_error(void);
int nmodl_abi_version(void);
int nmodl_device_count(int *out);
int nmodl_set_device(int dev);
int nmodl_get_device(int *dev);
int nmodl_device_info(int dev, int *sm_count, long long *l2_bytes, long long *mem_bytes,
                      int *cc_major, int *cc_minor, char *name, int name_len);
int nmodl_malloc(void **out, size_t bytes);
int nmodl_free(void *p);
int nmodl_host_alloc(void **out, size_t bytes);
int nmodl_host_free(void *p);
int nmodl_host_register(void *p, size_t bytes);
int nmodl_host_unregister(void *p);
int nmodl_memcpy_h2d(void *dst, const void *src, size_t bytes, nmodl_stream_t s);
int nmodl_memcpy_d2h(void *dst, const void *src, size_t bytes, nmodl_stream_t s);
int nmodl_memcpy_d2d(void *dst, const void *src, size_t bytes, nmodl_stream_t s);
int nmodl_memset(void *dst, int value, size_t bytes, nmodl_stream_t s);
int nmodl_stream_create(nmodl_stream_t *out);
int nmodl_stream_destroy(nmodl_stream_t s);
int nmodl_stream_sync(nmodl_stream_t s);
int nmodl_device_sync(void);
int nmodl_event_create(nmodl_event_t *out);
int nmodl_event_destroy(nmodl_event_t e);
int nmodl_event_record(nmodl_event_t e, nmodl_stream_t s);
int nmodl_stream_wait_event(nmodl_stream_t s, nmodl_event_t e);
/* event record that stays a timestamped node inside a stream capture
 * (cudaEventRecordExternal): kernel boundaries inside a replayed graph */
int nmodl_event_record_external(nmodl_event_t e, nmodl_stream_t s);
/* fold the currents of up to 8 one-instance-per-node populations (run with
 * seg_unique = 2, i.e. without their own node update) into node rhs/d, in
 * population order: rhs[node_index[j]] -= i_p[j], d[...] += g_p[j] */
int nmodl_combine_unique(double *rhs, double *d, const int *node_index, long long n,
                         const double *const *i_ptrs, const double *const *g_ptrs, int n_pops, nmodl_stream_t s);
/* the same fold; flags bit 0: launched for programmatic dependent launch
 * behind the kernel before it on the stream -- the population currents are
 * loaded at once, node rhs/d only after that kernel completes (it must not
 * write any i_p/g_p array) */
int nmodl_combine_unique_ex(double *rhs, double *d, const int *node_index, long long n,
                            const double *const *i_ptrs, const double *const *g_ptrs, int n_pops, int flags,
                            nmodl_stream_t s);
int nmodl_event_sync(nmodl_event_t e);
int nmodl_event_elapsed_ms(nmodl_event_t a, nmodl_event_t b, float *ms);
/* CUDA-graph capture of the per-timestep launch loop */
int nmodl_capture_begin(nmodl_stream_t s);
int nmodl_capture_end(nmodl_stream_t s, nmodl_graph_t *out);
/* upload the graph to the device before its first (timed) launch */
int nmodl_graph_upload(nmodl_graph_t g, nmodl_stream_t s);
int nmodl_graph_launch(nmodl_graph_t g, nmodl_stream_t s);
int nmodl_graph_destroy(nmodl_graph_t g);
/* status block */
int nmodl_status_reset(nmodl_status *st_dev, nmodl_stream_t s);
int nmodl_status_size(void);
/* first non-finite index of an array (atomicMin into *out_dev); the upload
 * half of the reference's whole-store scan, interp.py:538-545 */
int nmodl_first_nonfinite(const double *p, long long n, unsigned long long *out_dev, nmodl_stream_t s);
/* deterministic sum and sum|x| for cross-rank validation checksums */
int nmodl_checksum(const double *p, long long n, double *scratch_dev, double *out_dev, nmodl_stream_t s);
/* write a buffer larger than L2 (timing hygiene) */
int nmodl_l2_flush(double *buf, long long n_doubles, nmodl_stream_t s);
/* read a (zeroed) buffer larger than L2: cleans L2 after nmodl_l2_flush */
int nmodl_l2_clean(const double *buf, long long n_doubles, nmodl_stream_t s);
/* keep the stream busy for `ns` nanoseconds (one spinning thread) so host-issued
 * timed launches queue up behind it instead of leaving gaps in the timing */
int nmodl_spin(long long ns, nmodl_stream_t s);
/* node_index scatter layout: stable sort by node (perm, rank = perm^-1),
 * per-node counts and offsets.  Builder-defined extension: the reference has
 * no node arrays; the SIMD backend only marks ATOMIC_ADD,
 * codegen.py:77-78. */
int nmodl_scatter_layout(const int *node_index_dev, long long n, int n_nodes, unsigned int *counts_dev,
                         long long *offsets_dev, long long *scratch_dev, long long *perm_dev,
                         long long *rank_dev, int *bad_dev, nmodl_stream_t s);
/* occupied node segments (seg_node, seg_off = offsets[seg_node] ++ [n]) and
 * CTA tiles of whole segments, ~`tile` instances each; counts_dev[0] =
 * n_segs, counts_dev[1] = tile boundaries (n_tiles + 1).  Builder-defined. */
int nmodl_node_segments(const long long *offsets_dev, int n_nodes, long long n, long long tile,
                        int *seg_node_dev, long long *seg_off_dev, long long *tiles_dev, long long *counts_dev,
                        nmodl_stream_t s);
int nmodl_permute(const double *src, double *dst, const long long *perm, long long n, int inverse,
                  nmodl_stream_t s);
int nmodl_permute_i32(const int *src, int *dst, const long long *perm, long long n, nmodl_stream_t s);
int nmodl_gather_v(const double *node_v, const int *node_index, double *v, long long n, nmodl_stream_t s);
/* self-test: out_a[i] = nmodl::exp_c(x[i]), out_b[i] = exp(x[i]) (bit-equality check) */
int nmodl_selftest_exp(const double *x, double *out_a, double *out_b, long long n, nmodl_stream_t s);
/* self-test: out[i] = nmodl::div_a(a[i], b[i]) (relaxed division, CudaOptions.div_approx);
 * a signalling-NaN marker where the branch-free form disagrees without flagging */
int nmodl_selftest_div_approx(const double *a, const double *b, double *out, long long n, nmodl_stream_t s);
/* self-test: out[i] = nmodl::exp16(x[i]) (shared-memory table exp, CudaOptions.exp_smem);
 * flag[i] bit 0 = fast form flagged, bit 1 = fast and safe forms disagree without a flag */
int nmodl_selftest_exp_smem(const double *x, double *out, unsigned *flag, long long n, nmodl_stream_t s);

/* ---- NCCL: validation collectives only (no exchange on the per-step path) --
 * libnccl.so.2 is opened at first use; the unique id travels between the
 * ranks of one node through the caller's bootstrap (parallel.py: a file).
 * Replaces torch.distributed in the multi-GPU plumbing (PAPER.md:674-678:
 * one rank per device, instances sharded by cell). */
int nmodl_nccl_unique_id(unsigned char *out128);
int nmodl_nccl_init(void **comm, int nranks, const unsigned char *id128, int rank);
int nmodl_nccl_destroy(void *comm);
/* op: 0 = sum, 1 = max */
int nmodl_nccl_allreduce_f64(void *comm, const double *send, double *recv, long long count, int op,
                             nmodl_stream_t s);
int nmodl_nccl_allgather_f64(void *comm, const double *send, double *recv, long long count, nmodl_stream_t s);

/* ---- per-mechanism library (lib<mech>-<hash>.so) -----------------------
 * Every generated mechanism exports exactly these symbols.  `md` points to a
 * host copy of the mechanism's `<mech>_data` struct (device pointers inside);
 * `nsteps` launches are enqueued on `s`; flags bit 0 selects the
 * finite-difference Newton Jacobian (Runner(jac_mode="fd"), interp.py:127-131).
 *
 *   <mech>_initialize      replaces <mech>_initialize(md)      codegen.py:450-455
 *   <mech>_state_update    replaces <mech>_state_update(md)    codegen.py:450-455
 *   <mech>_current_update  replaces <mech>_current_update(md)  codegen.py:320-352
 *                          (writes i_acc/g_acc with zero-then-accumulate
 *                           semantics of interp.py:475-476; no memset needed)
 *   <mech>_step            fused state_update + current_update per timestep
 *                          (the interp.simulate inner loop, interp.py:650-652)
 *   <mech>_step_nodes      same, with v gathered through node_index and i/g
 *                          reduced into node rhs/d in instance order
 *   <mech>_abi             JSON description of <mech>_data (field order)
 *   <mech>_abi_size        sizeof(<mech>_data)
 *   <mech>_step_unique     (pipelined builds) step_nodes for one instance per
 *                          node: cp.async pipeline, no segment reduction
 *   <mech>_step_nodes_ctas resident CTAs of the node kernel on the current
 *                          device (the host sizes node tiles to whole waves)
 */
#define NMODL_B200_MECHANISM(mech)                                                    \
  int mech##_initialize(const void *md, int nsteps, nmodl_stream_t s, int flags);     \
  int mech##_state_update(const void *md, int nsteps, nmodl_stream_t s, int flags);   \
  int mech##_current_update(const void *md, int nsteps, nmodl_stream_t s, int flags); \
  int mech##_step(const void *md, int nsteps, nmodl_stream_t s, int flags);           \
  int mech##_step_nodes(const void *md, int nsteps, nmodl_stream_t s, int flags);     \
  const char *mech##_abi(void);                                                       \
  long long mech##_abi_size(void);                                                    \
  int mech##_step_nodes_ctas(void);

/* ---- population group library (libgroup_<name>-<hash>.so) -------------
 * Several one-instance-per-node populations stepped by one launch
 * (codegen_cuda.emit_group; an extension -- the reference steps one
 * mechanism per call, interp.py:456-471).  `a` points to a host copy of
 * `<name>_args`: the members' <mech>_data structs back to back, then
 * `long long cta[n_chains + 1]` (chain c owns CTAs [cta[c], cta[c+1])).
 *
 *   <name>_step_unique     `nsteps` group launches on `s` (0 or cudaError_t)
 *   <name>_step_group      same for a direct group (kind="direct": every CTA
 *                          runs every member in turn), <name>_group_ctas()
 *                          its resident CTAs
 *   <name>_args_size       sizeof(<name>_args)
 */
#define NMODL_B200_GROUP(name)                                                        \
  int name##_step_unique(const void *a, int nsteps, nmodl_stream_t s, int flags);     \
  long long name##_args_size(void);

#ifdef __cplusplus
}
#endif

#endif /* NMODL_B200_H */
