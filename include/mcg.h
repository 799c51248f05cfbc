/*
 * mcg.h — C ABI of the B200-native progressive material cache path
 * (arXiv 2305.07238 hot path: per-sample material-network evaluation with
 * progressive caching of cacheable-node outputs in an Nc x Ne two-hash table).
 *
 * Plain C: pointers, sizes and status codes; no C++ or torch types cross this
 * boundary. Every entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core). The reference throws C++
 * exceptions; here every call returns an mcg_status and leaves a thread-local
 * message in mcg_last_error(). The C++ drop-in shim maps the
 * codes back to the reference exception types:
 *
 *   MCG_ERR_INVALID_ARGUMENT -> std::invalid_argument   (cache.cpp:84-86, tracer.hpp:78)
 *   MCG_ERR_OVERFLOW         -> std::overflow_error     (cache.cpp:76-78)
 *   MCG_ERR_GRAPH            -> matcache::GraphError    (graph.hpp:89-96)
 *   MCG_ERR_COMPILE          -> matcache::CompileError  (stackvm.hpp:65-68)
 *   MCG_ERR_SCENE            -> matcache::SceneError    (scene.hpp:66-69)
 *   MCG_ERR_IMAGE_IO         -> matcache::ImageIoError  (image.hpp:24-27)
 *   MCG_ERR_IO               -> std::runtime_error      (cache.cpp:161, 172)
 *   MCG_ERR_CUDA / MCG_ERR_NO_DEVICE -> std::runtime_error (no reference analogue)
 *
 * Threading: a context owns one device and one CUDA stream; calls on one
 * context must be serialised by the caller (the reference render() is
 * synchronous too, tracer.hpp:69). Host-only calls (scene load, compile,
 * audit) are thread-safe on distinct objects.
 */
#ifndef MCG_H_
#define MCG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCG_ABI_VERSION 4   /* 2: mcg_render_stats.shadow_occluded; 3: write_slots, insert log, n_devices; 4: mcg_shadow_tree */

typedef enum mcg_status {
    MCG_OK = 0,
    MCG_ERR_INVALID_ARGUMENT = 1,
    MCG_ERR_OVERFLOW = 2,
    MCG_ERR_GRAPH = 3,
    MCG_ERR_COMPILE = 4,
    MCG_ERR_SCENE = 5,
    MCG_ERR_IMAGE_IO = 6,
    MCG_ERR_IO = 7,
    MCG_ERR_CUDA = 8,
    MCG_ERR_NO_DEVICE = 9
} mcg_status;

/* Message of the last failed call on this thread ("" after success). */
const char* mcg_last_error(void);
int mcg_abi_version(void);

/* ------------------------------------------------------------------------ */
/* Cache descriptor, hashes, codec (include/matcache/cache.hpp)             */
/* ------------------------------------------------------------------------ */

/* Layout-identical to matcache::CacheDescriptor (cache.hpp:17-25): 20 bytes,
 * mip_level at offset 8 followed by 3 padding bytes. */
typedef struct mcg_descriptor {
    uint32_t mat_idx;
    uint32_t node_idx;
    uint8_t mip_level;
    uint8_t pad_[3];
    uint32_t texel_x;
    uint32_t texel_y;
} mcg_descriptor;

/* Insert outcomes; values follow matcache::InsertOutcome (cache.hpp:51-56). */
enum { MCG_INSERT_WON = 0, MCG_INSERT_LOST_RACE = 1, MCG_INSERT_ALREADY_PRESENT = 2,
       MCG_INSERT_CELL_FULL = 3 };

/* Host (CPU) reference-identical scalar helpers, for tools and tests.
 * mcg_hash_cell/check: cache.cpp:34-39; codec: cache.cpp:41-71;
 * mcg_memory_bytes: cache.cpp:73-80 (returns MCG_ERR_OVERFLOW on overflow). */
uint64_t mcg_hash_cell(const mcg_descriptor* d);
uint32_t mcg_hash_check(const mcg_descriptor* d);
uint32_t mcg_encode_value(const float rgb[3]);
void mcg_decode_value(uint32_t packed, float rgb_out[3]);
mcg_status mcg_memory_bytes(uint64_t n_cells, uint64_t n_entries, uint64_t* bytes_out);

/* ------------------------------------------------------------------------ */
/* Device context                                                           */
/* ------------------------------------------------------------------------ */

typedef struct mcg_ctx mcg_ctx;

typedef struct mcg_options {
    int32_t device;       /* CUDA ordinal */
    int32_t profile;      /* 1: time every kernel launch with CUDA events on the ctx stream */
    void* stream;         /* optional cudaStream_t to use; NULL: the context creates its own */
    /* In-process multi-GPU (render() uses every worker, tracer.hpp:12, 69-70):
     * n_devices > 1 makes the context span `devices` (NULL: `device`,
     * device+1, ...; the first is the context's own). mcg_upload_scene
     * uploads to every device; mcg_render splits the image into 16x16 tiles
     * dealt round-robin to the devices (shard_mode 0, or contiguous bands
     * with shard_mode 1), one host thread and stream per device, each with
     * its own cache replica (the context's table on that device; an
     * external cache is refused), and gathers the frames on the first
     * device with ncclReduce(sum) of frames zeroed outside each device's
     * tiles (exact: x + 0 = x). A device listed twice (tests on one GPU)
     * gathers by device copies instead of NCCL. 0 or 1: one device. */
    int32_t n_devices;
    const int32_t* devices;
} mcg_options;

mcg_status mcg_create(const mcg_options* opt, mcg_ctx** out);
/* Number of visible CUDA devices (MCG_ERR_NO_DEVICE when there is none). */
mcg_status mcg_device_count(int32_t* count);
mcg_status mcg_destroy(mcg_ctx* ctx);
mcg_status mcg_synchronize(mcg_ctx* ctx);
/* The cudaStream_t the context launches on (for external event timing). */
void* mcg_stream(mcg_ctx* ctx);

/* Per-kernel device-time accounting (enabled by mcg_options.profile). Each
 * record: a kernel name, launch count and summed CUDA-event milliseconds,
 * plus the algorithmic bytes the launches moved. */
typedef struct mcg_kernel_time {
    char name[48];
    uint64_t launches;
    double ms;
    double algorithmic_bytes;
} mcg_kernel_time;
mcg_status mcg_kernel_times(mcg_ctx* ctx, mcg_kernel_time* out, int32_t cap, int32_t* n_out);
mcg_status mcg_kernel_times_reset(mcg_ctx* ctx);
/* Number of this library's kernels launched since the last reset. */
uint64_t mcg_launch_count(mcg_ctx* ctx);

/* Batched device evaluation of the descriptor pipeline (host buffers in/out).
 * hash: cache.cpp:21-39; codec: cache.cpp:41-71; mip/texel: raycone.cpp:67-83. */
mcg_status mcg_hash_batch(mcg_ctx* ctx, const mcg_descriptor* d, size_t n, uint64_t* cell_hash,
                          uint32_t* check);
mcg_status mcg_encode_batch(mcg_ctx* ctx, const float* rgb, size_t n, uint32_t* packed);
mcg_status mcg_decode_batch(mcg_ctx* ctx, const uint32_t* packed, size_t n, float* rgb);
mcg_status mcg_mip_texel_batch(mcg_ctx* ctx, const float* uv, const float* g1, const float* g2,
                               size_t n, int32_t mip_offset, uint8_t* mip, uint32_t* texel_xy);

/* ------------------------------------------------------------------------ */
/* Material cache table in HBM (cache.hpp:69-115)                            */
/* ------------------------------------------------------------------------ */

typedef struct mcg_cache mcg_cache;

typedef struct mcg_cache_counters {          /* MaterialCache::Counters, cache.hpp:92-97 */
    uint64_t lookups, hits, inserts_won, inserts_lost_full;
} mcg_cache_counters;

/* MaterialCache(n_cells, n_entries), cache.cpp:82-92: zeroed table; nonzero
 * sizes (MCG_ERR_INVALID_ARGUMENT) and no 64-bit overflow (MCG_ERR_OVERFLOW). */
mcg_status mcg_cache_create(mcg_ctx* ctx, uint64_t n_cells, uint32_t n_entries, mcg_cache** out);
mcg_status mcg_cache_destroy(mcg_cache* cache);
mcg_status mcg_cache_clear(mcg_cache* cache);          /* all slots empty, counters 0 */
mcg_status mcg_cache_shape(const mcg_cache* cache, uint64_t* n_cells, uint32_t* n_entries);

/* Batch update/lookup. MCG_APPLY_CONCURRENT: every element probes/CASes at
 * once (cache.cpp:94-119 semantics under a race: single CAS, LostRace drops).
 * MCG_APPLY_ORDERED: elements are applied as if one thread called update()
 * in array order (the deterministic-insert rule: lowest index wins).
 * outcome/slot/packed are UpdateResult (cache.hpp:58-62); any may be NULL. */
enum { MCG_APPLY_CONCURRENT = 0, MCG_APPLY_ORDERED = 1 };
mcg_status mcg_cache_update_batch(mcg_cache* cache, const mcg_descriptor* d, const float* rgb,
                                  size_t n, int32_t apply_mode, uint8_t* outcome, uint64_t* slot,
                                  uint64_t* packed);
/* MaterialCache::lookup, cache.cpp:121-136: hit[i] = 1 and rgb[3i..] decoded on a hit. */
mcg_status mcg_cache_lookup_batch(mcg_cache* cache, const mcg_descriptor* d, size_t n,
                                  uint8_t* hit, float* rgb);
/* Same two operations on device-resident arrays (no copies; stream-ordered). */
mcg_status mcg_cache_update_device(mcg_cache* cache, const mcg_descriptor* d_desc,
                                   const float* d_rgb, size_t n, int32_t apply_mode,
                                   uint8_t* d_outcome);
mcg_status mcg_cache_lookup_device(mcg_cache* cache, const mcg_descriptor* d_desc, size_t n,
                                   uint8_t* d_hit, float* d_rgb);

/* slot_word (cache.hpp:83-86) for [first, first+n); occupied_slots (cache.cpp:138-144). */
mcg_status mcg_cache_read_slots(mcg_cache* cache, uint64_t first, size_t n, uint64_t* words);
/* The inverse, host words -> slots [first, first+n): seeds a device table
 * from a host MaterialCache's slot_word()s (the drop-in render's external
 * cache, cache.hpp:83-86); no counters change. */
mcg_status mcg_cache_write_slots(mcg_cache* cache, uint64_t first, size_t n, const uint64_t* words);
mcg_status mcg_cache_occupied(mcg_cache* cache, uint64_t* occupied);
mcg_status mcg_cache_counters_get(mcg_cache* cache, mcg_cache_counters* out);
mcg_status mcg_cache_counters_reset(mcg_cache* cache);
/* dump (cache.cpp:159-173): u64 n_cells, u64 n_entries, then every slot word, LE. */
mcg_status mcg_cache_dump(mcg_cache* cache, const char* path);
/* Device pointer of the slot array, for tooling. Layout: a head array of
 * n_cells x min(n_entries, 8) words (a cell's first slots, one 64-byte DRAM
 * block), then a tail array of n_cells x (n_entries - 8) words when
 * n_entries > 8. Slot indices everywhere else in this API are the logical
 * cell * n_entries + entry. */
uint64_t* mcg_cache_device_slots(mcg_cache* cache);

/* Striped shared table (one logical Nc x Ne table over `world`
 * GPUs instead of per-GPU replicas). The stripe of `rank` holds the cells c
 * with c % world == rank (local cell c / world); lookups, inserts and renders
 * address any cell through the stripes' device pointers -- peers' over
 * NVLink (CUDA IPC within a node), or other stripes of the same process
 * (mcg_cache_attach_local, which also emulates a striped table on one GPU).
 * Hashing, cell and entry indices are the logical table's, so results equal
 * those of one Nc x Ne table; cross-process deterministic mode is not
 * provided (each process applies its own ordered stores). read_slots,
 * occupied and clear act on this stripe's words; dump needs world == 1. */
mcg_status mcg_cache_create_stripe(mcg_ctx* ctx, uint64_t n_cells, uint32_t n_entries, uint32_t rank,
                                   uint32_t world, mcg_cache** out);
mcg_status mcg_cache_attach_local(mcg_cache* cache, mcg_cache* const* stripes, uint32_t world);
mcg_status mcg_cache_ipc_handle(mcg_cache* cache, void* out, size_t cap);   /* 64 bytes */
mcg_status mcg_cache_attach_ipc(mcg_cache* cache, const void* handles, uint32_t world);
mcg_status mcg_cache_stripe_info(const mcg_cache* cache, uint32_t* rank, uint32_t* world,
                                 uint64_t* local_cells);

/* audit_dump (cache.cpp:175-230), host only. */
typedef struct mcg_audit_report {
    uint64_t n_cells, n_entries, occupied;
    int32_t clean;
    int64_t bad_cell;
    char problem[160];
} mcg_audit_report;
mcg_status mcg_audit_dump(const char* path, mcg_audit_report* out);

/* Descriptor trace (SURVEY §8d "replay a descriptor trace dumped from a
 * render"): while recording, every CacheLookup the VM makes through this
 * table (renders, mcg_execute_batch) appends its descriptor, in lookup order
 * (warp-aggregated), up to `capacity` records; stop returns the count kept.
 * mcg_probe_replay runs a descriptor list (host) through the table as the VM
 * would -- lookup, insert on a miss -- with the warp-cooperative probe, and
 * returns the device time, the algorithmic bytes and the outcome counts
 * (blocks_per_sm < 0: |blocks_per_sm| blocks per SM, software-pipelined,
 * for A/B runs). */
mcg_status mcg_cache_trace_start(mcg_cache* cache, uint64_t capacity);
mcg_status mcg_cache_trace_stop(mcg_cache* cache, uint64_t* recorded);
mcg_status mcg_cache_trace_read(mcg_cache* cache, uint64_t first, size_t n, mcg_descriptor* out);
mcg_status mcg_probe_replay(mcg_cache* cache, const mcg_descriptor* d, uint64_t n, int32_t blocks_per_sm,
                            double* ms, double* bytes, mcg_cache_counters* counters);

/* Won-insert log: while recording, every insert this table wins in a
 * concurrent-mode render (the VM's CacheStore) or a concurrent batch update
 * appends (descriptor, entry within its cell, payload), up to `capacity`
 * records (a table can win at most its empty-slot count). stop returns the
 * number won (> capacity: the log overflowed). Replaying the records through
 * MaterialCache::update (cache.cpp:94-119) in (cell, entry) order rebuilds
 * the device's inserts word for word in a host table that held the same
 * words before -- the drop-in render uses this to keep the caller's
 * external cache current. */
typedef struct mcg_insert_record {
    mcg_descriptor desc;
    uint32_t entry;
    uint32_t payload;
} mcg_insert_record;
mcg_status mcg_cache_insert_log_start(mcg_cache* cache, uint64_t capacity);
mcg_status mcg_cache_insert_log_stop(mcg_cache* cache, uint64_t* won);
mcg_status mcg_cache_insert_log_read(mcg_cache* cache, uint64_t first, size_t n, mcg_insert_record* out);

/* Probe microbenchmark: n descriptors generated on the device
 * from `seed` (mat<8, node<256, mip<=16, texel uniform in 2^mip), then one
 * phase over them: 0 insert-all, 1 lookup-all, 2 50/50 mix; phase + 16*v
 * selects the probe variant v: 0 two-round per-lane scan (first 16 B, then
 * the rest), 1 one-round per-lane scan (whole cell), 2 warp-cooperative
 * (coalesced whole cells + ballots; Ne = 10 only), 4 warp-cooperative with
 * 16-byte lanes (one round trip per probe; Ne even <= 10); 5 / 6 / 7 the same
 * probe software-pipelined over 2 / 4 / 1 batches of 32 descriptors per warp
 * (all head loads of the step in flight while the next step is hashed);
 * 10 / 11 as 7 / 5 with each lane scanning its own cell after a shared-memory
 * transpose of the warp's loads (fewer instructions than per-round ballots);
 * + 256*b runs b blocks of 256 threads per SM (default 8). Returns the kernel's
 * device milliseconds and the algorithmic bytes it moved. */
mcg_status mcg_probe_bench(mcg_cache* cache, uint64_t n, uint64_t seed, int32_t phase,
                           int32_t iters, double* ms_out, double* algorithmic_bytes_out);

/* ------------------------------------------------------------------------ */
/* Scenes and compiled materials (scene.hpp, graph.hpp, stackvm.hpp)         */
/* ------------------------------------------------------------------------ */

/* Opcode numbering == matcache::Opcode (stackvm.hpp:13-36). */
enum {
    MCG_OP_PUSH_CONST = 0, MCG_OP_LOAD_UV, MCG_OP_LOAD_POSITION, MCG_OP_LOAD_NORMAL,
    MCG_OP_LOAD_INCOMING, MCG_OP_TEX_SAMPLE, MCG_OP_CHECKER, MCG_OP_NOISE, MCG_OP_ADD,
    MCG_OP_SUB, MCG_OP_MUL, MCG_OP_DIV, MCG_OP_MIX, MCG_OP_CLAMP, MCG_OP_DOT, MCG_OP_SIN_WAVE,
    MCG_OP_RAMP, MCG_OP_POWER, MCG_OP_BSDF_DIFFUSE, MCG_OP_CACHE_LOOKUP, MCG_OP_CACHE_STORE,
    MCG_OP_END
};

/* mcg_insn.flags */
#define MCG_F_USES_UV 0x01u        /* cache ops: Instruction::uses_uv */
#define MCG_F_SCALAR_RESULT 0x02u  /* CacheLookup: Instruction::scalar_result */
#define MCG_F_WRAP_CLAMP 0x04u     /* TexSample: WrapMode::Clamp (else Repeat) */
#define MCG_F_UV_SHIFT 3           /* LoadUv: UvChannel in bits 3-4 (0 uv, 1 u, 2 v) */
/* mcg_insn.tags: static scalar tag of the operands/result */
#define MCG_T_A 0x01u   /* first (deepest) operand is scalar */
#define MCG_T_B 0x02u   /* second operand is scalar */
#define MCG_T_C 0x04u   /* third operand (Mix factor) is scalar */
#define MCG_T_R 0x08u   /* result is scalar */

/* One flattened instruction (16 B): matcache::Instruction (stackvm.hpp:40-54)
 * minus the host texture pointer, plus the compiler's static stack depth
 * `sp` (operand-stack depth before the instruction on the miss path) and the
 * static scalar tags. arg: PushConst -> const pool index; TexSample -> texture
 * id; Noise -> noise pool index; Ramp -> ramp index; cache ops -> node_idx.
 * imm: Checker scale (f) or CacheLookup skip_offset (i). store_ord: rank of a
 * CacheStore among the program's stores (deterministic-insert key). */
typedef struct mcg_insn {
    uint8_t op, flags, sp, tags;
    uint32_t arg;
    uint16_t bracket;
    uint8_t store_ord;
    uint8_t pad_;
    union {
        float f;
        int32_t i;
    } imm;
} mcg_insn;

typedef struct mcg_program {      /* CompiledProgram, stackvm.hpp:73-79 */
    uint32_t material_id;
    uint32_t code_offset, code_len;   /* into mcg_flat_scene.code */
    uint32_t max_stack;
    uint32_t cache_point_count;
} mcg_program;

typedef struct mcg_const { float v[3]; uint32_t scalar; } mcg_const;           /* Value */
typedef struct mcg_noise { int32_t octaves; float frequency, lacunarity, gain; } mcg_noise;
typedef struct mcg_ramp { uint32_t first, count; } mcg_ramp;
typedef struct mcg_ramp_stop { float t, r, g, b; } mcg_ramp_stop;            /* ops::RampStop */
typedef struct mcg_texture { int32_t width, height; uint64_t offset; } mcg_texture;

/* BVH node (32 B). Internal: a = left child, b = right child (both >= 0).
 * Leaf: a = ~first (negative), b = count; prims [first, first+count) of the
 * leaf-ordered primitive arrays. Same tree as Scene::build_bvh (scene.cpp:154-194). */
typedef struct mcg_bvh_node { float lo[3]; int32_t a; float hi[3]; int32_t b; } mcg_bvh_node;

#define MCG_PRIM_SPHERE 0x80000000u

typedef struct mcg_point_light { float position[3], intensity[3]; } mcg_point_light;
typedef struct mcg_rect_light { float corner[3], edge_u[3], edge_v[3], radiance[3]; } mcg_rect_light;

/* The prepared scene in the device layout (host pointers; owned by the
 * mcg_scene it came from). Primitives are stored in BVH leaf order
 * (Scene::prim_order_). prim_geom: 12 floats per prim; triangle:
 * p0.xyz,0, e1.xyz,0, e2.xyz,0 with e1 = p1-p0, e2 = p2-p0 (scene.cpp:61-62);
 * sphere: center.xyz, radius, 0... prim_uv: uv0,uv1,uv2 (6 floats).
 * prim_info: material slot | MCG_PRIM_SPHERE. */
typedef struct mcg_flat_scene {
    float cam_position[3], cam_look_at[3], cam_up[3];
    float cam_vfov_deg;
    int32_t cam_width, cam_height;
    float env[3];

    uint32_t n_prims;
    const float* prim_geom;
    const float* prim_uv;
    const uint32_t* prim_info;
    uint32_t n_nodes;
    const mcg_bvh_node* nodes;

    uint32_t n_point_lights, n_rect_lights;
    const mcg_point_light* point_lights;
    const mcg_rect_light* rect_lights;

    uint32_t n_programs;
    const mcg_program* programs;     /* indexed by material slot */
    uint32_t n_code;
    const mcg_insn* code;
    uint32_t n_consts;
    const mcg_const* consts;
    uint32_t n_noise;
    const mcg_noise* noise;
    uint32_t n_ramps;
    const mcg_ramp* ramps;
    uint32_t n_ramp_stops;
    const mcg_ramp_stop* ramp_stops;
    uint32_t n_textures;
    const mcg_texture* textures;
    uint64_t n_texels;
    const float* texels;             /* RGBA float4 per texel (A = 0), 16-B aligned */
} mcg_flat_scene;

typedef struct mcg_scene mcg_scene;

/* load_scene (scene.cpp:300-387): scene JSON + material JSON files + PPM
 * textures -> load_graph (graph.cpp:242) -> analyze (analysis.cpp:141) ->
 * compile (stackvm.cpp:210) -> prepare/build_bvh (scene.cpp:98, 154).
 * min_subtree_size: AnalysisOptions (analysis.hpp:36-40); pass 3 for default. */
mcg_status mcg_scene_load(const char* path, int32_t min_subtree_size, mcg_scene** out);
mcg_status mcg_scene_destroy(mcg_scene* scene);
mcg_status mcg_scene_flat(const mcg_scene* scene, mcg_flat_scene* out);
/* disassemble(program) (stackvm.cpp:370-443), same text, for material slot. */
mcg_status mcg_scene_disassemble(const mcg_scene* scene, uint32_t slot, char* buf, size_t cap,
                                 size_t* len_out);
/* analysis_to_json (analysis.cpp:160-184) for material slot. */
mcg_status mcg_scene_analysis_json(const mcg_scene* scene, uint32_t slot, char* buf, size_t cap,
                                   size_t* len_out);

/* Building blocks for a caller that already holds the reference's in-memory
 * types (the C++ drop-in shim): geometry in mesh form plus already-compiled
 * programs; the library builds the BVH (scene.cpp:98-194) and the flat layout. */
typedef struct mcg_mesh_in {
    uint32_t n_vertices, n_indices, material_id;
    const float* positions;   /* 3 per vertex */
    const float* uvs;         /* 2 per vertex */
    const uint32_t* indices;
} mcg_mesh_in;
typedef struct mcg_sphere_in { float center[3]; float radius; uint32_t material_id; } mcg_sphere_in;
typedef struct mcg_scene_in {
    float cam_position[3], cam_look_at[3], cam_up[3];
    float cam_vfov_deg;
    int32_t cam_width, cam_height;
    float env[3];
    uint32_t n_meshes, n_spheres;
    const mcg_mesh_in* meshes;
    const mcg_sphere_in* spheres;
    uint32_t n_point_lights, n_rect_lights;
    const mcg_point_light* point_lights;
    const mcg_rect_light* rect_lights;
    /* programs, already flattened by the caller (code/consts/... as in mcg_flat_scene) */
    uint32_t n_programs;
    const mcg_program* programs;
    uint32_t n_code;
    const mcg_insn* code;
    uint32_t n_consts;
    const mcg_const* consts;
    uint32_t n_noise;
    const mcg_noise* noise;
    uint32_t n_ramps;
    const mcg_ramp* ramps;
    uint32_t n_ramp_stops;
    const mcg_ramp_stop* ramp_stops;
    uint32_t n_textures;
    const mcg_texture* textures;
    uint64_t n_texels;
    const float* texels;
} mcg_scene_in;
mcg_status mcg_scene_build(const mcg_scene_in* in, mcg_scene** out);

/* Static stack schedule of one flattened program: fills sp / tags / store_ord
 * of every instruction and returns the miss-path stack bound, with compile()'s
 * balance checks and errors (stackvm.cpp:226-245 -> MCG_ERR_COMPILE). For
 * callers that flatten a reference CompiledProgram themselves. PushConst
 * args index `consts`. */
mcg_status mcg_schedule_program(mcg_insn* code, uint32_t n_code, const mcg_const* consts,
                                uint32_t n_consts, uint32_t* max_stack);

/* ------------------------------------------------------------------------ */
/* Rendering (tracer.hpp:7-70; body restated in DESIGN.md §render)           */
/* ------------------------------------------------------------------------ */

enum { MCG_CACHE_OFF = 0, MCG_CACHE_CONCURRENT = 1, MCG_CACHE_DETERMINISTIC = 2 };
enum { MCG_SHARD_INTERLEAVED = 0, MCG_SHARD_BANDS = 1 };

typedef struct mcg_render_params {   /* RenderConfig, tracer.hpp:7-20 */
    int32_t width, height;           /* 0 = camera's */
    int32_t spp, max_bounces;
    int32_t cache_mode;              /* MCG_CACHE_*; OFF == !cache_enabled */
    int32_t mip_offset;
    uint64_t n_cells;                /* used when no external cache is passed */
    uint32_t n_entries;
    uint32_t first_sample;           /* progressive renders: samples [first, first+spp) */
    uint64_t rng_seed;
    float diffuse_spread;
    int32_t tile_size;
    int32_t shard_rank, shard_count, shard_mode;   /* tile sharding across GPUs */
    int32_t samples_per_pass;        /* samples in flight per wavefront (0 = auto); in
                                        deterministic mode an insert epoch is one
                                        (pass, bounce) wavefront */
} mcg_render_params;

typedef struct mcg_frame {           /* FrameBuffers, tracer.hpp:24-43 (W*H pixels) */
    double* radiance;                /* 3 per pixel, row-major, row 0 at the top */
    double* nodes_found;             /* 1 per pixel */
    uint32_t* samples;               /* 1 per pixel */
} mcg_frame;

typedef struct mcg_render_stats {    /* RenderStats, tracer.hpp:45-55 */
    double wall_time_s;
    double device_ms;
    uint64_t lookups, hits, inserts_won, inserts_lost_full;
    uint64_t stores_attempted, stores_won, instructions_executed;
    uint64_t max_stack_seen;
    uint64_t paths, shading_points, shadow_rays;
    uint64_t bvh_nodes, prims_tested, tex_samples;   /* work counters (roofline bytes) */
    uint64_t bvh_nodes_shadow, prims_tested_shadow;  /* of which any-hit (shadow) rays */
    uint64_t closest_rays;                           /* continuation rays traced (after the primary) */
    uint64_t shadow_occluded;                        /* shadow rays that found an occluder */
    uint64_t launches;               /* this library's kernel launches in the call */
    uint64_t* hits_per_sample;       /* optional, caller array of spp entries */
} mcg_render_stats;

/* Make `scene` the context's current scene (uploads geometry, BVH, bytecode,
 * textures to HBM). */
mcg_status mcg_upload_scene(mcg_ctx* ctx, const mcg_scene* scene);

/* render(scene, config, external_cache) (tracer.hpp:69-70) on the uploaded
 * scene. cache: external table (NULL -> a context-owned table of
 * n_cells x n_entries, cleared for this call, as tracer.hpp:67-68 says).
 * mcg_render: host frame buffers (accumulated into: callers zero them for a
 * fresh render; copies are inside the call). mcg_render_device: frame
 * pointers are device memory (accumulated into), no host copies. */
mcg_status mcg_render(mcg_ctx* ctx, const mcg_render_params* params, mcg_cache* cache,
                      mcg_frame* frame, mcg_render_stats* stats);
mcg_status mcg_render_device(mcg_ctx* ctx, const mcg_render_params* params, mcg_cache* cache,
                             mcg_frame* d_frame, mcg_render_stats* stats);

/* Camera set-up shared by every implementation of render(): basis, tan of
 * the half field of view and the primary cone spread (cone_for_camera,
 * raycone.cpp:8-13). out: fwd[3], right[3], up[3], tan_half, aspect, spread. */
mcg_status mcg_camera_setup(const mcg_flat_scene* scene, int32_t width, int32_t height,
                            float out[12]);

/* Scene queries on the uploaded scene for a batch of rays (host buffers):
 * Scene::intersect (scene.cpp:252-278) -> 24 floats per ray (found, t,
 * position, normal, uv, slot, e1, e2, duv1, duv2; zeros on a miss) and
 * Scene::occluded (scene.cpp:280-298) -> 1 byte per ray, t_max per ray.
 * rays: 6 floats (origin, direction). variant selects the traversal the
 * renderer can use: 0 per-thread DFS over the reference's nodes,
 * 1 warp-synchronous child pairs, 2 4-wide, 3 speculative 4-wide (default),
 * 4 warp packets over the 4-wide tree; occluded also 5: speculative 4-wide over
 * a SAH hierarchy of the reference's leaves (the renderer's shadow rays).
 * Every variant returns the reference's answer. */
mcg_status mcg_intersect_batch(mcg_ctx* ctx, const float* rays, size_t n, float t_min, float t_max,
                               int32_t variant, float* out);
mcg_status mcg_occluded_batch(mcg_ctx* ctx, const float* rays, size_t n, float t_min,
                              const float* t_max, int32_t variant, uint8_t* out);

/* The any-hit (shadow) hierarchy of the uploaded scene, as built (on the
 * device by default; MCG_SHADOW_BUILD=host at upload: the host builder):
 * *n_out 4-wide nodes of mcg_bvh_node entries (leaf: a = ~first, b = count
 * with the reference leaf's exact box; node: a = index, b = -1; unused:
 * b = 0) copied to out when cap >= *n_out * 4, and the root entry. No
 * reference counterpart (the reference traces shadow rays over its own
 * tree, scene.cpp:280-298); for tests and tools. */
mcg_status mcg_shadow_tree(mcg_ctx* ctx, mcg_bvh_node* out, size_t cap, size_t* n_out, int32_t* root_a,
                           int32_t* root_b);

/* Per-shading-point material evaluation (execute, stackvm.cpp:248-368) on the
 * device for a batch of shading points of one material slot of the uploaded
 * scene. sp: 15 floats per point (position, normal, incoming, uv, g1, g2).
 * cache_mode: MCG_CACHE_OFF (or cache NULL) disables the binding;
 * MCG_CACHE_CONCURRENT stores with immediate CAS; MCG_CACHE_DETERMINISTIC
 * looks up against the table as it was at the call and applies the stores
 * afterwards in (point index, store ordinal) order. values: 3 floats + 1 tag
 * word (1 = scalar) per point; nodes_found / instructions per point
 * (EvalStats, stackvm.hpp:88-103). */
mcg_status mcg_execute_batch(mcg_ctx* ctx, uint32_t slot, const float* sp, size_t n,
                             mcg_cache* cache, int32_t cache_mode, int32_t mip_offset,
                             float* values, uint32_t* nodes_found, uint32_t* instructions);

#ifdef __cplusplus
}
#endif

#endif /* MCG_H_ */
