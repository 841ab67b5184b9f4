/* C-ABI of the B200 component-aware branch-and-reduce vertex-cover solver.
 *
 * Plain pointers and sizes only.  Every entry point returns 0 on success and
 * a nonzero code on failure, with vcg_last_error() describing it.  The
 * library never falls back to a CPU path: without a CUDA device every
 * compute entry point fails with VCG_ENODEV.
 *
 * Reference interfaces replaced (arxiv/paper_2512_18334 = python package
 * `vcsolver`, /root/reference/pkg/src/vcsolver):
 *   vcg_graph_create / vcg_graph_destroy  <- graph.py:74 build_csr / graph.py:33 StaticGraph
 *                                            (the CSR is uploaded once to HBM)
 *   vcg_induced_subgraph                   <- graph.py:99 induced_subgraph
 *   vcg_greedy_bound                       <- preprocess.py:28 greedy_bound
 *                                            (kernels/pure.py:306 greedy_cover)
 *   vcg_root_reduce                        <- preprocess.py:77 root_reduce
 *                                            (reductions.py:110 reduce_to_fixpoint
 *                                            + reductions.py:263 crown_reduce
 *                                            + graph.py:99 induced_subgraph)
 *   vcg_search                             <- engine.py:160 _Engine.run (the
 *                                            threaded search behind solve(),
 *                                            engine.py:561)
 *   vcg_crown_reduce                       <- reductions.py:263 crown_reduce
 *                                            (one crown on a node's degrees)
 *   vcg_node_op                            <- kernels/__init__.py:33-44, the
 *                                            per-node kernel API (pure.py /
 *                                            _native.pyx), one node per call
 *   vcg_brute_force_mvc                    <- oracle.py:28 brute_force_mvc
 *   vcg_registry_*                         <- registry.py:79-224 Registry (the
 *                                            search's device registry protocol,
 *                                            one operation per call or per thread)
 */
#ifndef VCGPU_H
#define VCGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VCG_OK 0
#define VCG_EINVAL 1
#define VCG_ENODEV 2
#define VCG_ECUDA 3
#define VCG_ERESOURCE 4
#define VCG_EPROTOCOL 5

typedef struct vcg_graph vcg_graph;

/* Upload a canonical CSR (offsets int64[n+1], neighbors int32[offsets[n]],
 * sorted slices, symmetric) to the current device. */
int vcg_graph_create(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                     vcg_graph** out);
/* Same, without copying the host arrays: the graph keeps pointers to
 * `offsets` / `neighbors` as its host view (the root pipeline's host-side
 * crown and greedy read them), so the caller must keep both alive and
 * unchanged until vcg_graph_destroy.  Uploads from pinned buffers run at
 * full PCIe speed.  (graph.py:33 StaticGraph: the Python mirror passes its
 * own arrays and holds them for the handle's lifetime.) */
int vcg_graph_create_borrowed(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                              vcg_graph** out);
int vcg_graph_destroy(vcg_graph* g);
int64_t vcg_graph_num_vertices(const vcg_graph* g);
int64_t vcg_graph_num_edges(const vcg_graph* g);
/* Copy the device CSR back (offsets int64[n+1], neighbors int32[2m]). */
int vcg_graph_download(const vcg_graph* g, int64_t* offsets, int32_t* neighbors);

/* Subgraph induced on keep[0..nkeep) (strictly increasing ids), built on the
 * device by flag / scan / gather.  vertex_map == keep. */
int vcg_induced_subgraph(const vcg_graph* g, const int64_t* keep, int64_t nkeep,
                         vcg_graph** out);

/* Max-degree greedy cover (lowest index on ties).  members may be NULL,
 * else receives the picks in order (capacity n). */
int vcg_greedy_bound(const vcg_graph* g, int32_t* members, int64_t* size);

/* One crown reduction (reductions.py:263 crown_reduce) on the live window
 * [lo, hi] of a node's degree array deg (uint32[n], updated in place: the
 * heads are removed).  heads (capacity n) receives the forced heads in
 * increasing order, indep (capacity n, may be NULL) the crown's independent
 * side in increasing order; *edges_removed the edges the heads took.  Both
 * counts are 0 when no crown exists.  Host C++ -- the same routine
 * vcg_root_reduce runs between its device fixpoint passes (a maximum
 * bipartite matching is a sequential augmenting-path search on a residual
 * that the device rules have already shrunk). */
int vcg_crown_reduce(int64_t n, const int64_t* offsets, const int32_t* neighbors, uint32_t* deg,
                     int64_t lo, int64_t hi, int32_t* heads, int64_t* nheads, int32_t* indep,
                     int64_t* nindep, int64_t* edges_removed);

typedef struct {
  int64_t n_reduced;
  int64_t m_reduced;
  int64_t forced_count;
  int64_t greedy_original;
  int64_t greedy_reduced;
  int64_t max_degree_reduced;
  int64_t rule_counts[4]; /* degree_one, degree_two_triangle, high_degree, crown */
  double seconds[3];      /* device reduction, crown, compaction */
  /* device time of the rule kernels (CUDA events on the calling thread's
   * stream), their launches, grid-wide scans of the degree array, and the
   * kernel kind (0 none, 1 single block on chip, 2 single block in HBM,
   * 3 grid-wide cooperative, 4 grid-wide frontier-driven: any-order callers) */
  double kernel_ms;
  int64_t kernel_launches;
  int64_t kernel_scans;
  int64_t kernel_kind;
  /* frontier kernel (kind 4): sweeps, adjacency entries walked, grid barriers */
  int64_t kernel_sweeps;
  int64_t kernel_walked;
  int64_t kernel_barriers;
  /* VCG_ROOT_LAZY_GREEDY: the smallest greedy_original under which the
   * speculative-budget rules equal the reference's (-1: no speculation) */
  int64_t spec_need;
} vcg_preprocessed;

/* `enabled` flags of vcg_root_reduce: bit 0 applies the rules; with
 * VCG_ROOT_ANY_ORDER the forced ids may come back in index order instead of
 * forcing order (same set and rule counts), which lets the device run the
 * fused order-free sweeps on an on-chip workspace (the solve path). */
#define VCG_ROOT_RULES 1
#define VCG_ROOT_ANY_ORDER 2
/* MVC without a bound (has_bound == 0): the greedy cover of g is not
 * computed (greedy_original = -1).  The rules run with the speculative budget
 * and report spec_need: the reduction equals the reference's iff the greedy
 * cover of g has >= spec_need vertices, which the caller certifies after the
 * search with the optimum it found (every cover, the greedy one included, has
 * >= optimum vertices), computing the greedy (vcg_greedy_bound) only when
 * optimum < spec_need, and rerunning with VCG_ROOT_NO_SPEC if the greedy is
 * below it too.  The search then starts from greedy_reduced (achieved): the
 * optimum is the same, only the search order can differ from the reference's
 * min(greedy_reduced, greedy_original - forced). */
#define VCG_ROOT_LAZY_GREEDY 4
/* Rules with the real MVC bound from the start (no speculation). */
#define VCG_ROOT_NO_SPEC 8

/* Root reduction (lightweight rules on the device to a joint fixpoint with
 * the crown rule) and device compaction of the survivors.
 * has_bound: 0 = no bound (MVC: the greedy cover of g is the bound),
 * 1 = `bound` given (PVC; greedy_original is not computed, reported as -1),
 * 2 = `bound` given and greedy_original computed as well.
 * forced_out: capacity n, original ids in forcing order (index order under
 * VCG_ROOT_ANY_ORDER); NULL keeps them on the device with the reduced graph
 * (vcg_graph_forced), which takes their download off the solve's path.
 * vertex_map_out: capacity n, reduced id -> original id.
 * reduced_out: new graph handle (the input handle itself is never aliased). */
int vcg_root_reduce(const vcg_graph* g, int enabled, int crown, int has_bound, int64_t bound,
                    vcg_preprocessed* info, int32_t* forced_out, int64_t* vertex_map_out,
                    vcg_graph** reduced_out);

/* The forced ids of the root reduction that produced `reduced` when it was
 * called with forced_out == NULL: *count of them, copied to out (capacity
 * *count, nullable). */
int vcg_graph_forced(const vcg_graph* reduced, int32_t* out, int64_t* count);

typedef struct {
  int width;                  /* 8, 16 or 32: degree-array entry width */
  int pvc;                    /* 0: MVC, 1: PVC with budget k_red */
  int64_t k_red;
  int64_t best_init;          /* root ChildEntry best */
  int best_init_achieved;
  int use_components;
  int use_bounds;
  int disable_pruning;
  int deterministic;          /* one worker, private stack only */
  int load_balance;           /* offload through the shared worklist */
  int workers;                /* persistent blocks; 0 = every resident slot */
  int threads;                /* block size; 0 = chosen from n */
  int64_t worklist_threshold; /* 0 = 2 * workers (engine.py:182) */
  double timeout;             /* seconds; 0 = none */
  int check_registry;         /* verify quiescence + conservation afterwards */
  int record_cover;           /* nodes carry cover bitsets; witnesses are recorded */
  int32_t* cover_out;         /* record_cover: receives a cover of the reduced graph
                                 (capacity n) whose size is <= best */
  const int32_t* root_deg;    /* NULL: search the whole graph.  Else the residual
                                 degree array (n entries) of a subtree root, e.g. one
                                 produced by vcg_expand; covers are counted from it */
  int warp_limit;             /* warp tier: subproblems with <= warp_limit (<= 128) live
                                 vertices are solved by one warp as bitmask tasks;
                                 0 = off, < 0 = auto (128 when the graph has <= 256
                                 vertices of average degree >= 8, else 64).  Ignored (off) in
                                 deterministic, record-cover, no-components and
                                 no-pruning runs. */
  int gpu_share;              /* concurrent searches sharing the device (>= 1): each
                                 takes 1/gpu_share of the resident block slots.  Calls
                                 from different host threads run concurrently (each
                                 thread has its own stream and pooled buffers). */
  int32_t* registry_out;      /* nullable: receives the registry after the search,
                                 entry i at [12 i, 12 i + 12): best key (2 best +
                                 !achieved), live count, link (parent / ancestor, -1 at
                                 the root), kind (0 child, 1 parent), sum, sum_achieved,
                                 initial_sum, folded_total, first_child, nchild,
                                 discovery_done, child_folded (registry.py:24-88) */
  int64_t registry_cap;       /* entries registry_out holds; a larger registry is not
                                 copied (registry_entries still reports its size) */
  struct vcg_exchange* exchange; /* nullable: in-flight bound / stop exchange with other
                                 searches (vcg_exchange_*); the kernel polls it and
                                 publishes its root scope's achieved best into it */
  struct vcg_peer* peer;      /* nullable: global best / stop words shared by every
                                 rank of a distributed solve (vcg_peer_*): the kernel
                                 reads them and updates them with system-scope atomics,
                                 no host in the loop */
  int64_t peer_offset;        /* cover size of this search's root in the global count
                                 (the subtree's S) */
} vcg_search_config;

typedef struct {
  int64_t best;               /* root scope best (reduced graph) */
  int best_achieved;
  int found;                  /* PVC: root best <= k_red was reached */
  int timed_out;
  int error;                  /* device-side error code (0 = none) */
  int64_t tree_nodes_visited;
  int64_t component_branches;
  int64_t worklist_pushes;
  int64_t worklist_pops;
  int64_t max_stack_depth;
  int64_t rule_counts[6];     /* degree_one, d2t, high_degree, crown, clique, cycle */
  int64_t registry_entries;
  int64_t registry_violations;
  double kernel_ms;           /* device time of the search kernel (CUDA events) */
  int workers;
  int threads;
  int64_t records_loaded;     /* node records read from HBM (stack + worklist pops) */
  int64_t records_stored;     /* node records written to HBM (children offloaded) */
  int64_t slot_bytes;         /* bytes per node record (32 B header + degree array) */
  int64_t phase_cycles[10];   /* SM cycles summed over blocks: idle, load, reduce, label,
                                 split, select, exclude, include, registry, other */
  int64_t cover_size;         /* record_cover: entries written to cover_out, -1 if the
                                 root's best has no recorded witness */
  int64_t fix_cycles[4];      /* fixpoint profile (thread-0 cycles): scans, degree-one, */
  int64_t fix_count[4];       /* triangle and high-degree sweeps, and their counts */
  int64_t warp_tasks;         /* warp-tier tasks solved */
  int64_t warp_nodes;         /* tree nodes processed by the warp tier (included in
                                 tree_nodes_visited) */
  int64_t warp_cycles;        /* SM cycles warps spent in warp-tier tasks */
  int warp_limit;             /* effective warp-tier size limit (0 = tier off) */
  int64_t warp_epoch_cycles;  /* block cycles (thread 0) in warp-tier epochs */
  int64_t warp_task_max_cycles; /* longest single warp task, SM cycles */
  int64_t trace[8];           /* ns after the search kernel started: last node-level
                                 step, first warp task start, last warp task end;
                                 then tree nodes and vertices of the longest warp task */
  int64_t kernel_t0_ns;       /* device %globaltimer when the search kernel started and */
  int64_t kernel_t1_ns;       /* when its drain finished (a timeline of concurrent solves) */
} vcg_search_result;

/* In-flight exchange between one running search and the rest of a
 * distributed solve (engine.py:453-495 semantics across processes / GPUs).
 * Three device words on the creating thread's current device: an external
 * bound for the search's root scope (a cover of that size exists elsewhere:
 * the root key is lowered to it, not achieved; <= 0 stops the search), an
 * external stop flag (PVC answered elsewhere), and the search's own best
 * achieved root cover, lowered by the kernel as it finds covers.  post / peek
 * are DMA copies on the calling thread's stream: another host thread may call
 * them while the search kernel runs (copy engines, no SM needed).  Replaces
 * the shared state of engine.py:200 _Engine (threads over one process). */
typedef struct vcg_exchange vcg_exchange;
int vcg_exchange_create(vcg_exchange** out);
int vcg_exchange_destroy(vcg_exchange* x);
/* reset: no external bound, no stop, no local best */
int vcg_exchange_reset(vcg_exchange* x);
/* bound < 0: leave the bound unchanged */
int vcg_exchange_post(vcg_exchange* x, int64_t bound, int stop);
/* the search's best achieved root cover so far (INT32_MAX: none) */
int vcg_exchange_peek(vcg_exchange* x, int64_t* local_best);

/* Peer words of a distributed solve: [best absolute cover, stop] in one
 * rank's device memory, mapped into the other ranks' processes by CUDA IPC
 * (over NVLink when the ranks are on different GPUs) so every running search
 * kernel reads the global best and publishes its own covers / the PVC stop
 * with system-scope atomics -- the device-side form of vcg_exchange, with no
 * host thread relaying.  create + handle on one rank, open on the others
 * (handle: VCG_PEER_HANDLE_BYTES opaque bytes); offer = atomic min / stop
 * from the host between searches; read = the current words. */
#define VCG_PEER_HANDLE_BYTES 64
typedef struct vcg_peer vcg_peer;
int vcg_peer_create(vcg_peer** out);
int vcg_peer_handle(const vcg_peer* p, void* handle);
int vcg_peer_open(const void* handle, vcg_peer** out);
int vcg_peer_destroy(vcg_peer* p);
int vcg_peer_offer(vcg_peer* p, int64_t best, int stop);
int vcg_peer_read(const vcg_peer* p, int64_t* best, int* stop);

/* Run the persistent search kernel.  hist_out (nullable, capacity n+2)
 * receives the components-per-branch histogram indexed by component count. */
int vcg_search(const vcg_graph* g, const vcg_search_config* cfg, vcg_search_result* res,
               int64_t* hist_out);

/* Breadth-first expansion of the root's search tree on the device (one
 * block), with the reference's node semantics (engine.py:277): reduce,
 * prune, leaf, or branch on the max-degree vertex; a node whose residual
 * graph is disconnected is not expanded (its subtree handles the split).
 * Stops once `target` open subtrees exist.  Each open subtree i gets its
 * cover-so-far sub_S[i] and residual degrees sub_deg[i*n .. i*n+n).
 * The subtrees partition the remaining search: MVC = min(best, min_i(sub_S[i]
 * + MVC(subtree i))) -- the unit of multi-GPU partitioning. */
typedef struct {
  int64_t target;
  int64_t best_init;          /* root scope bound, as for vcg_search */
  int use_components;
  int use_bounds;
} vcg_expand_config;

typedef struct {
  int64_t count;              /* open subtrees written */
  int64_t best;               /* best cover found by leaves during the expansion */
  int64_t nodes;              /* tree nodes processed by the expansion */
} vcg_expand_result;

int vcg_expand(const vcg_graph* g, const vcg_expand_config* cfg, vcg_expand_result* res,
               int32_t* sub_S, int32_t* sub_deg, int64_t capacity);

/* One per-node kernel on the device (parity surface of vcsolver.kernels).
 * op: 0 degree_one_pass, 1 degree_two_triangle_pass, 2 high_degree_pass,
 *     3 reduce_fixpoint, 4 recompute_bounds, 5 select_max_degree,
 *     6 count_live, 7 remove_vertex, 8 remove_neighbors,
 *     9 component of vertex `v` (bfs_component result set, index order),
 *     10 bfs_component (pure.py:258): out[0,n) = visited (in/out), out[n,2n) =
 *        the BFS queue, budget = stamp, v = source,
 *     11 next_live_unvisited (pure.py:297): out[0,n) = visited, budget =
 *        stamp, lo = start,
 *     12 greedy_cover (pure.py:306): picks to out[pos..], ret = {size, pos}
 * deg: host uint32[n] in/out.  out: host int32 (capacity 4n+4) in/out.
 * ret: host int64[8], op-specific (same tuples as the reference). */
int vcg_node_op(int op, int width, int64_t n, const int64_t* offsets, const int32_t* neighbors,
                uint32_t* deg, int64_t lo, int64_t hi, int64_t budget, int64_t v, int32_t* out,
                int64_t pos, int64_t* ret);

/* Exhaustive minimum vertex cover of a small graph (n <= 26), every vertex
 * subset checked on the device: *size = the minimum, witness (capacity n,
 * nullable) = the lexicographically smallest minimum cover in increasing
 * order (oracle.py:28 brute_force_mvc; n > 26 fails with VCG_EINVAL). */
int vcg_brute_force_mvc(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                        int64_t* size, int32_t* witness);

const char* vcg_last_error(void);
/* Number of kernels this library has launched so far (process-wide). */
int64_t vcg_launch_count(void);
int vcg_device_count(void);
/* Make `device` current for this thread's subsequent calls. */
int vcg_set_device(int device);
/* The calling thread's current device (-1 on error). */
int vcg_get_device(void);
/* Process teardown (call once, e.g. from atexit, after the calling program's
 * solver threads have finished): waits for the device, then turns every later
 * device-memory release into a no-op so that no CUDA call runs from static or
 * thread-local destructors while the runtimes unload.  No reference
 * counterpart (the reference holds no device state). */
void vcg_shutdown(void);

/* ------------------------------------------------ registry protocol --
 * registry.py:79-224 Registry as a device object: the search kernel's
 * registry arena (12 int32 fields per entry, the vcg_search registry_out row
 * layout) and its atomic encodings, one protocol operation per call.
 * Operations (a, b, c are the reference's arguments in order):
 *   NEW_CHILD        a = best_init (>= 1), b = parent (-1: none), c = achieved -> index
 *   NEW_PARENT       a = initial_sum (>= 0), b = ancestor                    -> index
 *   ATOMIC_MIN_BEST  a = candidate, b = achieved                    -> prior best
 *   BEST_SNAPSHOT                                   -> ret[0] best, ret[1] achieved
 *   INC/DEC_LIVE_NODES, INC/DEC_LIVE_COMPS                          -> new count
 *   ADD_TO_SUM       a = delta, b = achieved, c = folded            -> new sum
 *   MARK_DISCOVERY_DONE
 * Protocol violations return VCG_EPROTOCOL (registry.py:20
 * RegistryProtocolError): an increment on a finished entry is refused, a
 * decrement below zero stays applied. */
#define VCG_REG_NEW_CHILD 0
#define VCG_REG_NEW_PARENT 1
#define VCG_REG_ATOMIC_MIN_BEST 2
#define VCG_REG_BEST_SNAPSHOT 3
#define VCG_REG_INC_LIVE_NODES 4
#define VCG_REG_DEC_LIVE_NODES 5
#define VCG_REG_ADD_TO_SUM 6
#define VCG_REG_INC_LIVE_COMPS 7
#define VCG_REG_DEC_LIVE_COMPS 8
#define VCG_REG_MARK_DISCOVERY_DONE 9

typedef struct vcg_registry vcg_registry;
int vcg_registry_create(int64_t capacity, vcg_registry** out);
int vcg_registry_destroy(vcg_registry* r);
int64_t vcg_registry_size(const vcg_registry* r);
int vcg_registry_op(vcg_registry* r, int op, int64_t idx, int64_t a, int64_t b, int64_t c,
                    int64_t* ret /* [2] */);
/* count device threads at once: thread i runs `rounds` passes of
 * ops[0..nops) (nops <= 8, operations on existing entries) on entry idx[i]
 * with (a[i], b[i]) (a / b may be NULL: 0); ret[i] = its last result;
 * *protocol_error = the first violation code seen (0: none). */
int vcg_registry_concurrent(vcg_registry* r, const int* ops, int nops, int rounds,
                            const int64_t* idx, const int64_t* a, const int64_t* b,
                            int64_t count, int64_t* ret, int* protocol_error);
/* entries [0, *count) as 12-int32 rows (rows may be NULL to read the count) */
int vcg_registry_download(const vcg_registry* r, int32_t* rows, int64_t cap, int64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* VCGPU_H */
