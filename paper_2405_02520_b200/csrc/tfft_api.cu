// C ABI (include/tfft.h) of the B200 fault-tolerant FFT: plan objects,
// launch dispatch and the run_protected orchestration
// (reference abft/protected.py:63-166).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tfft.h"
#include "aux_kernels.cuh"
#include "fix.cuh"
#include "multi.cuh"
#include "registry.h"

using namespace tfft;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CU(call)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess)                                                     \
            return fail(TFFT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int ilog2(int64_t n) {
    int l = 0;
    while ((int64_t(1) << l) < n) ++l;
    return l;
}
bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

// exp(-2*pi*i*k/N) in long double with exact axis values and quadrant symmetry.
void unit_root(int64_t N, int64_t k, long double* re, long double* im) {
    k %= N;
    if (k < 0) k += N;
    const long double two_pi = 6.283185307179586476925286766559005768L;
    long double c, s;  // cos, sin of 2*pi*k/N
    if ((4 * k) % N == 0) {
        const int q = (int)((4 * k) / N);
        c = q == 0 ? 1.0L : (q == 2 ? -1.0L : 0.0L);
        s = q == 1 ? 1.0L : (q == 3 ? -1.0L : 0.0L);
    } else {
        const int64_t qn = N / 4;  // N >= 8 here
        const int q = (int)(k / qn);
        const int64_t r = k - q * qn;  // 0 < r < N/4
        long double c1, s1;
        if (2 * r <= qn) {
            c1 = cosl(two_pi * (long double)r / (long double)N);
            s1 = sinl(two_pi * (long double)r / (long double)N);
        } else {
            c1 = sinl(two_pi * (long double)(qn - r) / (long double)N);
            s1 = cosl(two_pi * (long double)(qn - r) / (long double)N);
        }
        switch (q) {
            case 0: c = c1; s = s1; break;
            case 1: c = -s1; s = c1; break;
            case 2: c = -c1; s = -s1; break;
            default: c = s1; s = -c1; break;
        }
    }
    *re = c;
    *im = -s;
}

// Multi-resolution root table of the Stockham engine: t[M + k] = w_M^k for
// every power of two 2 <= M <= L and k < M (engine.cuh), exactly rounded.
template <class T>
std::vector<C<T>> multires_table(int64_t L) {
    std::vector<C<T>> t(2 * L);
    t[0].x = t[1].x = (T)1;
    t[0].y = t[1].y = (T)0;
    for (int64_t M = 2; M <= L; M *= 2) {
        for (int64_t k = 0; k < M; ++k) {
            long double re, im;
            unit_root(M, k, &re, &im);
            t[M + k].x = (T)re;
            t[M + k].y = (T)im;
        }
    }
    return t;
}

struct Counters {
    int flag_count;
    int pad;
    unsigned long long max_key;  // float key in low 32 bits for fp32
    FixHead fix;                 // verdict header of the device-side correction (fix.cuh)
};
// Detection block: Counters (padded to 64 B), the device correction's
// per-job verdicts, then the flag records (64-byte aligned). One D2H copy of
// the first kBlockHead + kEarly records brings back everything a clean or a
// singly-faulted call needs.
constexpr size_t kFixOff = 64;
constexpr size_t kBlockHead = kFixOff + kFixCap * sizeof(FixRes);
static_assert(sizeof(Counters) <= kFixOff && kBlockHead % 64 == 0, "detection block layout");

// [prec][logn][variant] -> entry, plus the tuned default and a runtime override
constexpr int kMaxVariants = 32;
struct SingleIndex {
    const SingleEntry* e[2][14][kMaxVariants] = {};
    int count[2][14] = {};
    int chosen[2][14] = {};
    int override_[2][14];
    SingleIndex() {
        for (int p = 0; p < 2; ++p)
            for (int l = 0; l < 14; ++l) override_[p][l] = -1;
        for (int p = 0; p < 2; ++p) {
            const SingleTable* tabs = p == TFFT_FP32 ? kSingleTables_fp32 : kSingleTables_fp64;
            for (int part = 0; part < kSingleParts; ++part) {
                for (int i = 0; i < *tabs[part].count; ++i) {
                    const SingleEntry* en = &tabs[part].entries[i];
                    if (en->logn < 0 || en->logn >= 14 || en->variant >= kMaxVariants) continue;
                    e[p][en->logn][en->variant] = en;
                    count[p][en->logn] = std::max(count[p][en->logn], en->variant + 1);
                    if (en->chosen) chosen[p][en->logn] = en->variant;
                }
            }
        }
    }
};
SingleIndex& single_index() {
    static SingleIndex idx;
    return idx;
}

// The entry a launch uses: the runtime override (tuning) or the tuned default;
// table encodings are only instantiated on the default variant.
const SingleEntry* single_entry(int prec, int logn, int abft = 0) {
    if (logn < 0 || logn >= 14) return nullptr;
    SingleIndex& ix = single_index();
    const int ov = ix.override_[prec][logn];
    const SingleEntry* en = ix.e[prec][logn][ov >= 0 ? ov : ix.chosen[prec][logn]];
    if (en && !en->fn[abft]) en = ix.e[prec][logn][ix.chosen[prec][logn]];
    return en;
}

std::mutex g_attr_mu;
std::map<const void*, int> g_blocks_per_sm;

int prepare_kernel(const void* fn, int threads, int smem, int* blocks_per_sm) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_blocks_per_sm.find(fn);
    if (it != g_blocks_per_sm.end()) {
        *blocks_per_sm = it->second;
        return TFFT_OK;
    }
    // opt in always: static + dynamic shared memory may pass 48 KB together
    CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int nb = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem));
    if (nb < 1) return fail(TFFT_EUNSUPPORTED, "kernel does not fit on an SM");
    g_blocks_per_sm[fn] = nb;
    *blocks_per_sm = nb;
    return TFFT_OK;
}

}  // namespace

struct tfft_plan {
    int64_t n = 0;
    int prec = 0;
    int nstages = 0;
    int64_t dims[3] = {0, 0, 0};
    int64_t bs = 1;
    int device = 0;
    int check_level = 0;            // 0 threadblock checksums, 1 thread-level (scheme comparison)
    int dev_fix = 1;                // single-kernel sizes: correct on the device behind the launch
    int logn = 0;
    int num_sms = 148;
    size_t esize = 8;               // bytes per complex element
    // single-kernel path
    const SingleEntry* single = nullptr;
    void* tw = nullptr;             // w_N^k, k < N (single-kernel path)
    // multi-pass path
    MultiPlan multi;
    // Execution-only 3-pass split for large 2-stage plans (short L per pass;
    // the API plan's L = 1024..2048 passes read 32-64 B row segments). Used
    // whenever no stage:k hook coordinates are involved; the API plan keeps
    // execute_stage and stage faults. pass_count is the API plan's.
    MultiPlan fast;
    bool have_fast = false;
    // workspace
    Counters* d_cnt = nullptr;
    Counters* h_cnt = nullptr;      // pinned
    // the first kEarly flag entries ride back with the counters (pinned), so a
    // rare fault costs no extra host round trip before the decision
    static constexpr int kEarly = 64;
    unsigned char* h_block = nullptr;  // pinned: Counters (64 B) + kEarly FlagRec
    int64_t early_n = 0;
    unsigned char* d_block = nullptr;  // device: Counters (64 B) + FlagRec[flag_cap]
    FlagRec* d_flag_rec = nullptr;
    int64_t flag_cap = 0;           // records (bounded by kMaxFlagRecords)
    unsigned* d_ovf = nullptr;      // overflow bitmask, one bit per signal of the batch (zero between calls)
    int64_t ovf_bits = 0;
    // the last protected call's complete lists (tfft_report_fetch)
    std::vector<tfft_flag> last_flagged;
    std::vector<std::pair<int64_t, int64_t>> last_corrected;
    std::vector<int64_t> last_unrec;
    void* d_scratch = nullptr;      // correction staging
    size_t scratch_bytes = 0;
    FixJob* d_jobs = nullptr;
    int64_t jobs_cap = 0;
    void* d_ftab = nullptr;         // campaign fault table (single kernel)
    size_t ftab_bytes = 0;
    void* d_rel = nullptr;          // campaign per-signal rel discrepancies
    size_t rel_bytes = 0;
    cudaEvent_t ev_done = nullptr;  // detection summary landed in h_cnt
    // device-side correction off the caller's stream: the fix pass (latency
    // bound, ~10-50 us when something was flagged) overlaps whatever the
    // caller queues next; _finish orders the caller's stream behind it
    cudaStream_t s_fix = nullptr;
    cudaEvent_t ev_kern = nullptr;
    bool fix_side = false;
    // host-streaming path (tfft_run_protected_host): a ring of device chunk
    // buffers, copy streams for each direction, per-slot events
    static constexpr int kRing = 3;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    void* ring = nullptr;           // kRing x (in chunk, out chunk)
    size_t ring_chunk = 0;          // bytes of one chunk buffer
    cudaEvent_t ev_in[kRing] = {}, ev_comp[kRing] = {}, ev_out[kRing] = {};
    void* h_stage = nullptr;        // file path: pinned kRing x (in chunk, out chunk)
    size_t h_stage_chunk = 0;
};

namespace {

// The detection block: counters, then up to kMaxFlagRecords flag records;
// flags past that land in a per-signal overflow bitmask (batch / 8 bytes,
// written only in that degenerate case and cleared by read_summary).
constexpr int64_t kMaxFlagRecords = int64_t(1) << 16;
int ensure_flags(tfft_plan* p, int64_t batch) {
    const int64_t cap = std::max<int64_t>(std::min<int64_t>(batch, kMaxFlagRecords), tfft_plan::kEarly);
    if (cap > p->flag_cap || !p->d_block) {
        unsigned char* blk = nullptr;
        CU(cudaMalloc(&blk, kBlockHead + cap * sizeof(FlagRec)));
        CU(cudaMemset(blk, 0, kBlockHead));
        cudaFree(p->d_block);
        p->d_block = blk;
        p->d_cnt = reinterpret_cast<Counters*>(blk);
        p->d_flag_rec = reinterpret_cast<FlagRec*>(blk + kBlockHead);
        p->flag_cap = cap;
    }
    if (batch > p->flag_cap && batch > p->ovf_bits) {
        const int64_t bits = (batch + 31) / 32 * 32;
        unsigned* m = nullptr;
        CU(cudaMalloc(&m, bits / 8));
        CU(cudaMemset(m, 0, bits / 8));
        cudaFree(p->d_ovf);
        p->d_ovf = m;
        p->ovf_bits = bits;
    }
    return TFFT_OK;
}

int ensure_scratch(tfft_plan* p, size_t bytes) {
    if (bytes <= p->scratch_bytes) return TFFT_OK;
    cudaFree(p->d_scratch);
    p->d_scratch = nullptr;
    CU(cudaMalloc(&p->d_scratch, bytes));
    p->scratch_bytes = bytes;
    return TFFT_OK;
}

// Per-launch transform description shared by every path.
struct Launch {
    const void* in;
    void* out;
    int64_t batch;
    int64_t sig_base;
    int inverse;
    int scale_inv;
    int abft;              // ABFT_OFF / ABFT_WANG / ABFT_TABLE
    const void* etw;
    const void* values;
    double delta, abs_floor;
    // fault translated for this launch
    long long f_signal, f_elem;
    int f_where, f_stage, f_comp, f_bit;
    // batched campaign: one fault per f_div signals (device table for the
    // single kernel, host list for multi-pass) and per-signal rel output
    const FaultRec* f_table;
    const HostFault* faults;
    long long nfaults, f_div;
    void* rel_out;
};

// STAGE 5 tensor map: (batch x N) complex rows as 32-bit words; box of S rows
// x (N + pad) elements, pad = 32 B, so each row lands at a padded smem stride.
int encode_single_tmap(CUtensorMap* map, const void* base, int64_t n, int64_t batch, int esize, int S) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = [] {
        void* q = nullptr;
        cudaDriverEntryPointQueryResult r;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) != cudaSuccess ||
            r != cudaDriverEntryPointSuccess)
            return (EncodeFn) nullptr;
        return (EncodeFn)q;
    }();
    if (!fn) return fail(TFFT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t cw = esize / 4;
    cuuint64_t dims[2] = {cw * (cuuint64_t)n, (cuuint64_t)batch};
    cuuint64_t strides[1] = {(cuuint64_t)n * esize};
    cuuint32_t box[2] = {(cuuint32_t)(cw * (n + 32 / esize)), (cuuint32_t)S};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TFFT_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return TFFT_OK;
}

template <class T>
int launch_single_t(tfft_plan* p, const Launch& L, cudaStream_t st) {
    const SingleEntry* e = single_entry(p->prec, p->logn, L.abft);
    if (!e) return fail(TFFT_EUNSUPPORTED, "no single-kernel config");
    const void* fn = e->fn[L.abft];
    int nb = 0;
    int rc = prepare_kernel(fn, e->threads, e->smem, &nb);
    if (rc) return rc;
    SingleArgs<T> a;
    memset(&a, 0, sizeof(a));
    a.in = (const C<T>*)L.in;
    a.out = (C<T>*)L.out;
    a.batch = L.batch;
    a.sig_base = L.sig_base;
    a.tw = (const C<T>*)p->tw;
    a.etw = (const C<T>*)L.etw;
    a.values = (const C<T>*)L.values;
    a.delta = (T)L.delta;
    a.abs_floor = (T)L.abs_floor;
    a.floor_coef = p->prec == TFFT_FP32 ? (T)1e-6f : (T)1e-12;
    a.inverse = L.inverse;
    a.scale_inv = L.scale_inv;
    a.flag_count = &p->d_cnt->flag_count;
    a.flag_rec = p->d_flag_rec;
    a.flag_cap = p->flag_cap;
    a.flag_ovf = p->d_ovf;
    a.max_key = (typename KeyT<T>::type*)&p->d_cnt->max_key;
    a.rel_out = (T*)L.rel_out;
    a.f_table = L.f_table;
    a.f_div = L.f_div;
    a.f_signal = L.f_signal;
    a.f_elem = L.f_elem;
    a.f_where = L.f_where;
    a.f_comp = L.f_comp;
    a.f_bit = L.f_bit;
    const int S = e->threads / e->tps;
    const long long tiles = (L.batch + S - 1) / S;
    if ((e->stage & 7) == 5) {  // rows as a 2-D tensor, box padded past the signal end
        int rc2 = encode_single_tmap(&a.tmap, L.in, p->n, L.batch, (int)p->esize, S);
        if (rc2) return rc2;
    }
    long long grid = std::min<long long>(tiles, (long long)nb * p->num_sms);
    if (grid < 1) grid = 1;
    void* args[] = {&a};
    CU((tfft::note_launch(), cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(e->threads), args, e->smem, st)));
    return TFFT_OK;
}

int launch_transform(tfft_plan* p, const Launch& L, cudaStream_t st) {
    if (L.batch == 0) return TFFT_OK;
    if (p->single) {
        return p->prec == TFFT_FP32 ? launch_single_t<float>(p, L, st)
                                    : launch_single_t<double>(p, L, st);
    }
    MultiLaunch m;
    memset(&m, 0, sizeof(m));
    m.in = L.in; m.out = L.out; m.batch = L.batch; m.sig_base = L.sig_base;
    m.inverse = L.inverse; m.scale_inv = L.scale_inv; m.abft = L.abft;
    m.etw = L.etw; m.values = L.values; m.delta = L.delta; m.abs_floor = L.abs_floor;
    m.f_signal = L.f_signal; m.f_elem = L.f_elem; m.f_where = L.f_where;
    m.f_stage = L.f_stage; m.f_comp = L.f_comp; m.f_bit = L.f_bit;
    m.flag_count = &p->d_cnt->flag_count;
    m.flag_rec = p->d_flag_rec;
    m.flag_cap = p->flag_cap;
    m.flag_ovf = p->d_ovf;
    m.max_key = &p->d_cnt->max_key;
    m.only_stage = -1;
    m.faults = L.faults;
    m.nfaults = L.nfaults;
    m.f_div = L.f_div;
    m.rel_out = L.rel_out;
    bool api_layout = L.f_where == 2;  // a stage:k fault addresses the API plan's intermediates
    for (long long r = 0; L.faults && r < L.nfaults && !api_layout; ++r) api_layout = L.faults[r].where == 2;
    MultiPlan& mp = (p->have_fast && !api_layout) ? p->fast : p->multi;
    int rc = multi_launch(mp, m, st);
    if (rc) return fail(rc, multi_last_error());
    return TFFT_OK;
}

// The device-side correction pass (fix.cuh) of a single-kernel plan: plan
// mode (jobs == nullptr) right behind the fused launch, or list mode with
// host-chosen jobs. Returns TFFT_EUNSUPPORTED when the plan's kernel config
// has no fix instantiation (tuning overrides), so callers fall back.
template <class T>
int launch_fix_t(tfft_plan* p, const void* in, void* out, const void* etw, const void* values, double delta,
                 double abs_floor, int inverse, int one_sided, FixJob* jobs, int njobs, cudaStream_t st) {
    const SingleEntry* e = single_entry(p->prec, p->logn);
    if (!e || !e->fix) return TFFT_EUNSUPPORTED;
    int nb = 0;
    int rc = prepare_kernel(e->fix, e->fix_threads, e->fix_smem, &nb);
    if (rc) return rc;
    FixArgs<T> a;
    memset(&a, 0, sizeof(a));
    a.in = (const C<T>*)in;
    a.out = (C<T>*)out;
    a.bs = p->bs;
    a.tw = (const C<T>*)p->tw;
    a.etw = (const C<T>*)etw;
    a.values = (const C<T>*)values;
    a.delta = (T)delta;
    a.abs_floor = (T)abs_floor;
    a.floor_coef = p->prec == TFFT_FP32 ? (T)1e-6f : (T)1e-12;
    a.inverse = inverse;
    a.scale_inv = inverse;
    a.one_sided = one_sided;
    a.flag_count = &p->d_cnt->flag_count;
    a.flag_rec = p->d_flag_rec;
    a.jobs = jobs;
    a.njobs = njobs;
    a.jobs_out = jobs;
    a.head = &p->d_cnt->fix;
    a.res = reinterpret_cast<FixRes*>(p->d_block + kFixOff);
    const int grid = jobs ? std::max(1, std::min(njobs, 2 * p->num_sms)) : 8;
    void* args[] = {&a};
    CU((tfft::note_launch(), cudaLaunchKernel(e->fix, dim3(grid), dim3(e->fix_threads), args, e->fix_smem, st)));
    return TFFT_OK;
}

int launch_fix(tfft_plan* p, const void* in, void* out, const void* etw, const void* values, double delta,
               double abs_floor, int inverse, int one_sided, FixJob* jobs, int njobs, cudaStream_t st) {
    return p->prec == TFFT_FP32
               ? launch_fix_t<float>(p, in, out, etw, values, delta, abs_floor, inverse, one_sided, jobs, njobs, st)
               : launch_fix_t<double>(p, in, out, etw, values, delta, abs_floor, inverse, one_sided, jobs, njobs,
                                      st);
}

Launch base_launch(const void* in, void* out, int64_t batch, int inverse) {
    Launch L;
    memset(&L, 0, sizeof(L));
    L.in = in;
    L.out = out;
    L.batch = batch;
    L.inverse = inverse;
    L.scale_inv = inverse;
    L.abft = ABFT_OFF;
    L.f_where = AT_NONE;
    return L;
}

int check_plan(tfft_plan* p) {
    if (!p) return fail(TFFT_EINVAL, "null plan");
    CU(cudaSetDevice(p->device));
    return TFFT_OK;
}

// One fault in launch coordinates. Single-kernel plans: where is
// AT_INPUT / AT_PRESCALE / AT_OUTPUT and elem the natural-order element;
// multi-pass plans: where 1 input / 2 stage / 3 output with the reference
// layout index (translated per pass by multi_launch). where == AT_NONE: the
// fault never fires (outside the batch, or a `where` the reference never
// emits), like the reference's injector.
struct FaultT {
    long long signal = 0, elem = 0;
    int where = AT_NONE, stage = 0, comp = 0, bit = 0;
};

int translate_fault(const tfft_plan* p, const tfft_fault& f, int64_t batch, FaultT& out) {
    out = FaultT();
    if (f.where == TFFT_AT_NONE) return TFFT_OK;
    const int64_t n = p->n;
    const int width = p->prec == TFFT_FP32 ? 32 : 64;
    bool fires = f.signal >= 0 && f.signal < batch && f.element >= 0 && f.element < n;
    if (f.where == TFFT_AT_STAGE && (f.stage < 0 || f.stage >= p->nstages)) fires = false;
    if (f.where < TFFT_AT_NONE || f.where > TFFT_AT_OUTPUT) fires = false;
    if (!fires) return TFFT_OK;
    if (f.bit < 0 || f.bit >= width) return fail(TFFT_EINVAL, "bit out of range for the precision");
    if (f.component != 0 && f.component != 1) return fail(TFFT_EINVAL, "component must be re/im");
    out.signal = f.signal;
    out.comp = f.component;
    out.bit = f.bit;
    out.stage = f.stage;
    if (p->single) {
        if (f.where == TFFT_AT_INPUT) {
            out.where = AT_INPUT;
            out.elem = f.element;
        } else if (f.where == TFFT_AT_OUTPUT) {
            out.where = AT_OUTPUT;
            out.elem = f.element;
        } else {
            if (f.stage != p->nstages - 1)
                return fail(TFFT_EUNSUPPORTED, "intermediate-stage injection needs a multi-pass size");
            // last-stage hook index -> natural order
            const int64_t e = f.element;
            int64_t g = e;
            if (p->nstages == 2) {
                const int64_t d0 = p->dims[0], d1 = p->dims[1];
                g = (e / d1) + d0 * (e % d1);
            } else if (p->nstages == 3) {
                const int64_t d0 = p->dims[0], d1 = p->dims[1], d2 = p->dims[2];
                const int64_t k0 = e / (d1 * d2), k1 = (e / d2) % d1, k2 = e % d2;
                g = k0 + d0 * k1 + d0 * d1 * k2;
            }
            out.where = AT_PRESCALE;
            out.elem = g;
        }
    } else {
        out.where = f.where == TFFT_AT_INPUT ? 1 : (f.where == TFFT_AT_STAGE ? 2 : 3);
        out.elem = f.element;
    }
    return TFFT_OK;
}

// Copy streams, per-slot events and the device chunk ring of the streaming
// (host / file) paths.
int ensure_ring(tfft_plan* p, size_t chunk, cudaStream_t st) {
    if (!p->s_h2d) {
        CU(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
        for (int i = 0; i < tfft_plan::kRing; ++i) {
            CU(cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&p->ev_out[i], cudaEventDisableTiming));
        }
    }
    if (!p->ev_done) CU(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
    if (chunk > p->ring_chunk) {
        CU(cudaStreamSynchronize(st));
        CU(cudaStreamSynchronize(p->s_h2d));
        CU(cudaStreamSynchronize(p->s_d2h));
        cudaFree(p->ring);
        p->ring = nullptr;
        p->ring_chunk = 0;
        if (cudaMalloc(&p->ring, 2 * tfft_plan::kRing * chunk) != cudaSuccess)
            return fail(TFFT_ENOMEM, "host-streaming ring");
        p->ring_chunk = chunk;
    }
    return TFFT_OK;
}

// Whole checksum groups per streaming chunk: ~32 MiB, deep enough to hide
// launch gaps, small enough that pipeline fill/drain is a few percent of a
// 1 GiB batch.
int64_t groups_per_chunk(const tfft_plan* p, int64_t batch) {
    const int64_t grp_bytes = p->n * (int64_t)p->esize * p->bs;
    static const int64_t target = [] {
        const char* e = getenv("TFFT_STREAM_CHUNK_MB");  // tuning override
        const long long mb = e ? atoll(e) : 0;
        return mb > 0 ? (int64_t)mb << 20 : (int64_t)1 << 25;
    }();
    int64_t gpc = std::max<int64_t>(1, target / grp_bytes);
    return std::min<int64_t>(gpc, batch / p->bs);
}

// The detection summary behind the kernels: counters plus the first kEarly
// flag entries (only read on the host when flag_count says so), then ev_done.
int enqueue_summary(tfft_plan* p, cudaStream_t st) {
    // one copy: the counters and the first kEarly flag records
    p->early_n = std::min<int64_t>(tfft_plan::kEarly, p->flag_cap);
    CU(cudaMemcpyAsync(p->h_block, p->d_block, kBlockHead + p->early_n * sizeof(FlagRec), cudaMemcpyDeviceToHost,
                       st));
    if (!p->ev_done) CU(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
    CU(cudaEventRecord(p->ev_done, st));
    return TFFT_OK;
}

// Validation, report reset and the fault translated into launch coordinates
// (shared by the device and the host-streaming entry points).
int prepare_protected(tfft_plan* p, const void* in, void* out, int64_t batch, int scheme, double delta,
                      const void* etw, const void* values, double abs_floor, const tfft_fault* fault, int inverse,
                      tfft_report* rep, Launch& L) {
    if (!rep) return fail(TFFT_EINVAL, "null report");
    if (batch < 0 || (batch > 0 && (!in || !out))) return fail(TFFT_EINVAL, "batch must have shape (B, n) with n == plan.n");
    if (batch % p->bs) return fail(TFFT_EINVAL, "batch size not divisible by group size");
    if (scheme < TFFT_SCHEME_NONE || scheme > TFFT_SCHEME_TWO_SIDED_GROUP) return fail(TFFT_EINVAL, "bad scheme");
    const bool prot = scheme != TFFT_SCHEME_NONE;
    if (prot && !etw) return fail(TFFT_EINVAL, "protected schemes need the encoding row");
    if (prot && !(delta > 0)) return fail(TFFT_EINVAL, "delta must be positive");
    const int64_t groups = batch / p->bs;
    rep->groups = groups;
    rep->recompute_count = 0;
    rep->pass_count = 2 * (int64_t)p->nstages * groups;
    rep->max_rel_discrepancy = 0.0;
    rep->n_flagged = rep->n_corrected = rep->n_unrecoverable = 0;
    rep->fault_fired = 0;
    p->last_flagged.clear();
    p->last_corrected.clear();
    p->last_unrec.clear();

    L = base_launch(in, out, batch, inverse ? 1 : 0);
    L.abft = prot ? (values ? ABFT_TABLE : (p->check_level ? ABFT_THREAD : ABFT_WANG)) : ABFT_OFF;
    L.etw = etw;
    L.values = values;
    L.delta = delta;
    L.abs_floor = abs_floor;
    // ---- translate the fault into the launch's coordinates
    if (fault && fault->where != TFFT_AT_NONE) {
        FaultT ft;
        int rc = translate_fault(p, *fault, batch, ft);
        if (rc) return rc;
        if (ft.where != AT_NONE) {
            L.f_signal = ft.signal;
            L.f_elem = ft.elem;
            L.f_where = ft.where;
            L.f_stage = ft.stage;
            L.f_comp = ft.comp;
            L.f_bit = ft.bit;
            rep->fault_fired = 1;
        }
    }
    return TFFT_OK;
}

}  // namespace

extern "C" {

const char* tfft_last_error(void) { return g_err.c_str(); }

int tfft_tune_variants(int precision, int logn) {
    if ((precision != TFFT_FP32 && precision != TFFT_FP64) || logn < 1 || logn > 13) return 0;
    return single_index().count[precision][logn];
}

int tfft_tune_pass_variants(int precision, int logl) {
    if ((precision != TFFT_FP32 && precision != TFFT_FP64) || logl < 1 || logl >= 12) return 0;
    return pass_tune_variants(precision, logl);
}

int tfft_tune_pass_select(int precision, int logl, int kind, int variant) {
    int rc = pass_tune_select(precision, logl, kind, variant);
    if (rc) return fail(rc, multi_last_error());
    return TFFT_OK;
}

int tfft_tune_select(int precision, int logn, int variant) {
    if ((precision != TFFT_FP32 && precision != TFFT_FP64) || logn < 1 || logn > 13)
        return fail(TFFT_EINVAL, "no single-kernel size");
    SingleIndex& ix = single_index();
    if (variant >= ix.count[precision][logn] || (variant >= 0 && !ix.e[precision][logn][variant]))
        return fail(TFFT_EINVAL, "no such variant");
    ix.override_[precision][logn] = variant < 0 ? -1 : variant;
    return TFFT_OK;
}
int tfft_version(void) { return 1; }

int tfft_plan_create(tfft_plan** out, int64_t n, int precision, int nstages, const int64_t* dims,
                     int64_t bs, int device) {
    if (!out) return fail(TFFT_EINVAL, "null output handle");
    *out = nullptr;
    if (!is_pow2(n) || n < 2) return fail(TFFT_EINVAL, "n must be a power of two >= 2");
    if (precision != TFFT_FP32 && precision != TFFT_FP64) return fail(TFFT_EINVAL, "bad precision");
    if (nstages < 1 || nstages > 3 || !dims) return fail(TFFT_EINVAL, "plans use 1 to 3 stages");
    int64_t prod = 1;
    for (int i = 0; i < nstages; ++i) {
        if (!is_pow2(dims[i]) || dims[i] < 2) return fail(TFFT_EINVAL, "stage dims must be powers of two");
        prod *= dims[i];
    }
    if (prod != n) return fail(TFFT_EINVAL, "stage dims must multiply to n");
    if (bs < 1) return fail(TFFT_EINVAL, "bs must be >= 1");
    if (n > (int64_t(1) << 25)) return fail(TFFT_EUNSUPPORTED, "n above 2^25 not built");
    CU(cudaSetDevice(device));
    tfft_plan* p = new tfft_plan();
    p->n = n;
    p->prec = precision;
    p->nstages = nstages;
    for (int i = 0; i < nstages; ++i) p->dims[i] = dims[i];
    p->bs = bs;
    p->device = device;
    p->logn = ilog2(n);
    p->esize = precision == TFFT_FP32 ? 8 : 16;
    cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
    int rc = TFFT_OK;
    auto cleanup = [&](int code) {
        tfft_plan_destroy(p);
        return code;
    };
    if (p->logn <= 13) {
        p->single = single_entry(precision, p->logn);
        if (!p->single) return cleanup(fail(TFFT_EUNSUPPORTED, "no single-kernel config"));
        size_t bytes = (size_t)2 * n * p->esize;
        if (cudaMalloc(&p->tw, bytes) != cudaSuccess) return cleanup(fail(TFFT_ENOMEM, "twiddle alloc"));
        cudaError_t ce;
        if (precision == TFFT_FP32) {
            auto t = multires_table<float>(n);
            ce = cudaMemcpy(p->tw, t.data(), bytes, cudaMemcpyHostToDevice);
        } else {
            auto t = multires_table<double>(n);
            ce = cudaMemcpy(p->tw, t.data(), bytes, cudaMemcpyHostToDevice);
        }
        if (ce != cudaSuccess) return cleanup(fail(TFFT_ECUDA, cudaGetErrorString(ce)));
    } else {
        rc = multi_plan_init(p->multi, n, precision, nstages, dims, p->num_sms);
        if (rc) return cleanup(fail(rc, multi_last_error()));
        // measured crossover (profiles/sweep_r01_*): fp32 from 2^20, fp64 from 2^19
        static const int fast_env = [] {
            const char* e = getenv("TFFT_FAST3_MIN_LOGN");  // tuning override
            return e ? atoi(e) : 0;
        }();
        const int fast_min = fast_env ? fast_env : (precision == TFFT_FP32 ? 20 : 19);
        if (nstages == 2 && p->logn >= fast_min) {
            const int q = p->logn / 3, r = p->logn % 3;  // balanced, larger parts last
            int64_t d3[3];
            for (int i = 0; i < 3; ++i) d3[i] = int64_t(1) << (q + (i >= 3 - r ? 1 : 0));
            p->have_fast = multi_plan_init(p->fast, n, precision, 3, d3, p->num_sms) == TFFT_OK;
            if (!p->have_fast) multi_plan_free(p->fast);
        }
    }
    if (ensure_flags(p, tfft_plan::kEarly) != TFFT_OK) return cleanup(TFFT_ENOMEM);
    if (cudaMallocHost(&p->h_block, kBlockHead + tfft_plan::kEarly * sizeof(FlagRec)) != cudaSuccess)
        return cleanup(fail(TFFT_ENOMEM, "pinned detection block"));
    p->h_cnt = reinterpret_cast<Counters*>(p->h_block);
    *out = p;
    return TFFT_OK;
}

int tfft_plan_destroy(tfft_plan* p) {
    if (!p) return TFFT_OK;
    cudaSetDevice(p->device);
    cudaFree(p->tw);
    multi_plan_free(p->multi);
    if (p->have_fast) multi_plan_free(p->fast);
    cudaFree(p->d_block);
    cudaFree(p->d_ovf);
    if (p->h_block) cudaFreeHost(p->h_block);
    cudaFree(p->d_scratch);
    cudaFree(p->d_jobs);
    cudaFree(p->d_ftab);
    cudaFree(p->d_rel);
    if (p->ev_done) cudaEventDestroy(p->ev_done);
    if (p->ev_kern) cudaEventDestroy(p->ev_kern);
    if (p->s_fix) cudaStreamDestroy(p->s_fix);
    cudaFree(p->ring);
    if (p->h_stage) cudaFreeHost(p->h_stage);
    for (int i = 0; i < tfft_plan::kRing; ++i) {
        if (p->ev_in[i]) cudaEventDestroy(p->ev_in[i]);
        if (p->ev_comp[i]) cudaEventDestroy(p->ev_comp[i]);
        if (p->ev_out[i]) cudaEventDestroy(p->ev_out[i]);
    }
    if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
    if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
    delete p;
    return TFFT_OK;
}

int tfft_execute(tfft_plan* p, const void* in, void* out, int64_t batch, int inverse, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (batch < 0 || (batch > 0 && (!in || !out))) return fail(TFFT_EINVAL, "bad buffers");
    Launch L = base_launch(in, out, batch, inverse ? 1 : 0);
    return launch_transform(p, L, (cudaStream_t)stream);
}

int tfft_execute_stage(tfft_plan* p, int k, const void* in, void* out, int64_t batch, int inverse,
                       void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (batch < 0 || (batch > 0 && (!in || !out))) return fail(TFFT_EINVAL, "bad buffers");
    if (k < 0 || k >= p->nstages) return fail(TFFT_EINVAL, "stage index out of range");
    if (batch == 0) return TFFT_OK;
    if (p->single) {
        if (p->nstages != 1)
            return fail(TFFT_EUNSUPPORTED, "per-stage execution of a multi-stage plan needs n > 2^13");
        Launch L = base_launch(in, out, batch, inverse ? 1 : 0);
        L.scale_inv = 0;
        return launch_transform(p, L, (cudaStream_t)stream);
    }
    rc = multi_launch_stage(p->multi, k, in, out, batch, inverse ? 1 : 0, (cudaStream_t)stream);
    if (rc) return fail(rc, multi_last_error());
    return TFFT_OK;
}

int tfft_scale(void* buf, int64_t count, int dtype_bytes, double s, void* stream) {
    if (!buf || count < 0) return fail(TFFT_EINVAL, "bad buffer");
    if (dtype_bytes != 8 && dtype_bytes != 16) return fail(TFFT_EINVAL, "unsupported dtype");
    if (count == 0) return TFFT_OK;
    const int grid = (int)std::min<long long>((count + 255) / 256, 1 << 16);
    if (dtype_bytes == 8)
        tfft::note_launch(), scale_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>((float2*)buf, count, (float)s);
    else
        tfft::note_launch(), scale_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>((double2*)buf, count, s);
    CU(cudaGetLastError());
    return TFFT_OK;
}

int tfft_flip_bit(void* buf, int64_t word, int bit, int dtype_bytes, void* stream) {
    if (!buf || word < 0) return fail(TFFT_EINVAL, "bad buffer");
    const int wbytes = dtype_bytes / 2;
    if (wbytes != 4 && wbytes != 8) return fail(TFFT_EINVAL, "dtype must be complex64/complex128");
    if (bit < 0 || bit >= wbytes * 8) return fail(TFFT_EINVAL, "bit out of range");
    tfft::note_launch(), flip_word_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(buf, word, bit, wbytes);
    CU(cudaGetLastError());
    return TFFT_OK;
}

int tfft_encode_group(tfft_plan* p, const void* xg, int64_t bs, const void* row, void* s0, void* s1,
                      void* c_in, void* x_l1, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!xg || bs < 1) return fail(TFFT_EINVAL, "bad group");
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = p->n;
    if (s0 || s1) {
        int grid = (int)std::min<long long>((n + 255) / 256, 4LL * p->num_sms);
        if (p->prec == TFFT_FP32)
            tfft::note_launch(), group_sums_kernel<float><<<grid, 256, 0, st>>>((const float2*)xg, bs, n, (float2*)s0, (double2*)s1);
        else
            tfft::note_launch(), group_sums_kernel<double><<<grid, 256, 0, st>>>((const double2*)xg, bs, n, (double2*)s0, (double2*)s1);
        CU(cudaGetLastError());
    }
    if (c_in || x_l1) {
        if (p->prec == TFFT_FP32)
            tfft::note_launch(), dot_l1_kernel<float><<<(unsigned)bs, AUX_THREADS, 0, st>>>((const float2*)xg, n, (const float2*)row,
                                                                       (float2*)c_in, (float*)x_l1);
        else
            tfft::note_launch(), dot_l1_kernel<double><<<(unsigned)bs, AUX_THREADS, 0, st>>>((const double2*)xg, n, (const double2*)row,
                                                                        (double2*)c_in, (double*)x_l1);
        CU(cudaGetLastError());
    }
    return TFFT_OK;
}

int tfft_detect(tfft_plan* p, const void* yg, int64_t bs, const void* values, const void* c_in,
                const void* x_l1, double abs_floor, double floor_coef, void* rel, void* raw, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!yg || !c_in || !x_l1 || !rel || bs < 1) return fail(TFFT_EINVAL, "bad buffers");
    if (!(floor_coef >= 0)) return fail(TFFT_EINVAL, "floor_coef must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    if (p->prec == TFFT_FP32)
        tfft::note_launch(), detect_kernel<float><<<(unsigned)bs, AUX_THREADS, 0, st>>>(
            (const float2*)yg, p->n, (const float2*)values, (const float2*)c_in, (const float*)x_l1,
            (float)abs_floor, (float)floor_coef, (float*)rel, (float2*)raw);
    else
        tfft::note_launch(), detect_kernel<double><<<(unsigned)bs, AUX_THREADS, 0, st>>>(
            (const double2*)yg, p->n, (const double2*)values, (const double2*)c_in, (const double*)x_l1,
            abs_floor, floor_coef, (double*)rel, (double2*)raw);
    CU(cudaGetLastError());
    return TFFT_OK;
}

int tfft_correct_signal(tfft_plan* p, const void* s0, const void* yg, int64_t bs, int64_t f, void* fixed,
                        int inverse, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!s0 || !yg || !fixed || f < 0 || f >= bs) return fail(TFFT_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    rc = ensure_scratch(p, p->n * p->esize);
    if (rc) return rc;
    Launch L = base_launch(s0, p->d_scratch, 1, inverse ? 1 : 0);
    rc = launch_transform(p, L, st);
    if (rc) return rc;
    int grid = (int)std::min<long long>((p->n + 255) / 256, 4LL * p->num_sms);
    if (p->prec == TFFT_FP32)
        tfft::note_launch(), rebuild_kernel<float><<<grid, 256, 0, st>>>((const float2*)p->d_scratch, (const float2*)yg, bs, p->n, f,
                                                    (float2*)fixed);
    else
        tfft::note_launch(), rebuild_kernel<double><<<grid, 256, 0, st>>>((const double2*)p->d_scratch, (const double2*)yg, bs, p->n,
                                                     f, (double2*)fixed);
    CU(cudaGetLastError());
    return TFFT_OK;
}

int tfft_run_protected(tfft_plan* p, const void* in, void* out, int64_t batch, int scheme, double delta,
                       double abs_floor, const void* etw, const void* values, const tfft_fault* fault,
                       int inverse, tfft_report* rep, void* stream) {
    int rc = tfft_protect_launch(p, in, out, batch, scheme, delta, abs_floor, etw, values, fault, inverse, rep,
                                 stream);
    if (rc) return rc;
    return tfft_protect_finish(p, in, out, batch, scheme, delta, abs_floor, etw, values, inverse, rep, stream);
}

int tfft_protect_launch(tfft_plan* p, const void* in, void* out, int64_t batch, int scheme, double delta,
                        double abs_floor, const void* etw, const void* values, const tfft_fault* fault,
                        int inverse, tfft_report* rep, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Launch L;
    rc = prepare_protected(p, in, out, batch, scheme, delta, etw, values, abs_floor, fault, inverse, rep, L);
    if (rc) return rc;
    if (batch == 0) return TFFT_OK;  // an empty shard: empty report, nothing launched
    const bool prot = scheme != TFFT_SCHEME_NONE;
    if (prot) {
        rc = ensure_flags(p, batch);
        if (rc) return rc;
        CU(cudaMemsetAsync(p->d_cnt, 0, sizeof(Counters), st));
    }
    rc = launch_transform(p, L, st);
    if (rc) return rc;
    if (!prot) return TFFT_OK;
    // single-kernel sizes: the corrections run on the device right behind the
    // transform (fix.cuh), so the summary below already carries the verdicts.
    // The fix pass and the summary copy go to the plan's side stream (after
    // the transform): the caller's stream moves on to its next work at once.
    p->fix_side = false;
    cudaStream_t sum_st = st;
    if (p->single && p->dev_fix && scheme != TFFT_SCHEME_NONE) {
        if (!p->s_fix) CU(cudaStreamCreateWithFlags(&p->s_fix, cudaStreamNonBlocking));
        if (!p->ev_kern) CU(cudaEventCreateWithFlags(&p->ev_kern, cudaEventDisableTiming));
        CU(cudaEventRecord(p->ev_kern, st));
        CU(cudaStreamWaitEvent(p->s_fix, p->ev_kern, 0));
        rc = launch_fix(p, in, out, etw, values, delta, abs_floor, inverse ? 1 : 0,
                        scheme == TFFT_SCHEME_ONE_SIDED, nullptr, 0, p->s_fix);
        if (rc && rc != TFFT_EUNSUPPORTED) return rc;
        sum_st = p->s_fix;
        p->fix_side = true;
    }
    // the (tiny) detection summary rides back behind the transform
    rc = enqueue_summary(p, sum_st);
    if (rc) return rc;
    return TFFT_OK;
}

}  // extern "C"

namespace {

// Exact rel of `sigs` (indices into the device buffers in/out) for the
// signals the kernels sent back (recheck_kernel).
int recheck_device(tfft_plan* p, const void* in, const void* out, const std::vector<long long>& sigs,
                   const void* etw, const void* values, double abs_floor, std::vector<double>& rel,
                   cudaStream_t st) {
    rel.assign(sigs.size(), 0.0);
    if (sigs.empty()) return TFFT_OK;
    const size_t k = sigs.size();
    int rc = ensure_scratch(p, k * (sizeof(long long) + sizeof(double)));
    if (rc) return rc;
    long long* d_sig = (long long*)p->d_scratch;
    double* d_rel = (double*)(d_sig + k);
    CU(cudaMemcpyAsync(d_sig, sigs.data(), k * sizeof(long long), cudaMemcpyHostToDevice, st));
    if (p->prec == TFFT_FP32)
        tfft::note_launch(), recheck_kernel<float><<<(unsigned)k, AUX_THREADS, 0, st>>>(
            (const float2*)in, (const float2*)out, p->n, d_sig, (const float2*)etw, (const float2*)values,
            (float)abs_floor, 1e-6f, d_rel);
    else
        tfft::note_launch(), recheck_kernel<double><<<(unsigned)k, AUX_THREADS, 0, st>>>(
            (const double2*)in, (const double2*)out, p->n, d_sig, (const double2*)etw, (const double2*)values,
            abs_floor, 1e-12, d_rel);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(rel.data(), d_rel, k * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return TFFT_OK;
}

// Exact rel of host-resident signals `sg` (sorted global indices), staged
// through ring slot 0 in runs of consecutive signals (an all-zero batch flags
// every signal: one copy per run, one recheck launch per slot fill).
// `stage(first, count, din, dout)` copies the input / output rows of signals
// [first, first + count) into the device slot.
using StageFn = std::function<int(int64_t, int64_t, char*, char*)>;
int recheck_staged(tfft_plan* p, const std::vector<long long>& sg, std::vector<double>& rr, const void* etw,
                   const void* values, double abs_floor, const StageFn& stage, cudaStream_t st) {
    rr.assign(sg.size(), 0.0);
    const size_t sig_bytes = (size_t)p->n * p->esize;
    const int64_t cap = std::max<int64_t>(1, (int64_t)(p->ring_chunk / sig_bytes));
    char* din = (char*)p->ring;
    char* dout = din + p->ring_chunk;
    size_t i = 0;
    while (i < sg.size()) {
        std::vector<long long> local;
        const size_t i0 = i;
        int64_t used = 0;
        while (i < sg.size() && used < cap) {
            size_t j = i + 1;
            while (j < sg.size() && sg[j] == sg[j - 1] + 1 && used + (int64_t)(j - i) < cap) ++j;
            const int64_t cnt = (int64_t)(j - i);
            int rc = stage(sg[i], cnt, din + used * sig_bytes, dout + used * sig_bytes);
            if (rc) return rc;
            for (int64_t k = 0; k < cnt; ++k) local.push_back(used + k);
            used += cnt;
            i = j;
        }
        std::vector<double> r;
        int rc = recheck_device(p, din, dout, local, etw, values, abs_floor, r, st);
        if (rc) return rc;
        for (size_t k = 0; k < r.size(); ++k) rr[i0 + k] = r[k];
    }
    return TFFT_OK;
}

// Resolves the exact rel of recheck signals (global indices) -> rel.
using RecheckFn = std::function<int(const std::vector<long long>&, std::vector<double>&)>;

// Detection summary of the launches since the last counter reset: max rel
// discrepancy and the flagged (global signal, rel) list, sorted like the
// reference's group loop. Entries with the recheck sentinel (rel < 0) are
// resolved exactly through `resolve` and merged.
int read_summary(tfft_plan* p, int64_t batch, cudaStream_t st, tfft_report* rep,
                 std::vector<std::pair<long long, double>>& flags, double delta, const RecheckFn& resolve,
                 std::vector<std::pair<long long, double>>* rechecked = nullptr) {
    CU(cudaEventSynchronize(p->ev_done));
    const int64_t ntotal = std::min<int64_t>(p->h_cnt->flag_count, batch);
    const int64_t nflag = std::min<int64_t>(ntotal, p->flag_cap);
    double max_rel;
    if (p->prec == TFFT_FP32) {
        unsigned int k = (unsigned int)(p->h_cnt->max_key & 0xffffffffull);
        float f;
        memcpy(&f, &k, 4);
        max_rel = f;
    } else {
        memcpy(&max_rel, &p->h_cnt->max_key, 8);
    }
    flags.clear();
    std::vector<long long> rsig;
    if (nflag > 0 && nflag <= p->early_n) {  // already on the host
        const FlagRec* hr = reinterpret_cast<const FlagRec*>(p->h_block + kBlockHead);
        for (int64_t i = 0; i < nflag; ++i) {
            if (hr[i].rel < 0) rsig.push_back(hr[i].sig);
            else flags.emplace_back(hr[i].sig, hr[i].rel);
        }
    } else if (nflag > 0) {
        std::vector<FlagRec> recs(nflag);
        CU(cudaMemcpyAsync(recs.data(), p->d_flag_rec, nflag * sizeof(FlagRec), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        std::vector<long long> sig(nflag);
        std::vector<double> rel(nflag);
        for (int64_t i = 0; i < nflag; ++i) { sig[i] = recs[i].sig; rel[i] = recs[i].rel; }
        for (int64_t i = 0; i < nflag; ++i) {
            if (rel[i] < 0) rsig.push_back(sig[i]);
            else flags.emplace_back(sig[i], rel[i]);
        }
    }
    if (ntotal > nflag) {  // degenerate batch: the rest are bits of the overflow mask
        const int64_t words = (batch + 31) / 32;
        std::vector<unsigned> mask(words);
        CU(cudaMemcpyAsync(mask.data(), p->d_ovf, words * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CU(cudaMemsetAsync(p->d_ovf, 0, words * sizeof(unsigned), st));
        CU(cudaStreamSynchronize(st));
        for (int64_t w = 0; w < words; ++w)
            for (unsigned m = mask[w]; m; m &= m - 1) rsig.push_back(w * 32 + __builtin_ctz(m));
    }
    if (!rsig.empty()) {
        std::sort(rsig.begin(), rsig.end());
        std::vector<double> rr;
        int rc = resolve(rsig, rr);
        if (rc) return rc;
        for (size_t i = 0; i < rsig.size(); ++i) {
            const double r = rr[i];
            if (r > max_rel || r != r) max_rel = r != r ? INFINITY : r;
            const bool hit = p->prec == TFFT_FP32 ? (float)r > (float)delta : r > delta;
            if (hit) flags.emplace_back(rsig[i], r);
            if (rechecked) rechecked->emplace_back(rsig[i], r);
        }
    }
    std::sort(flags.begin(), flags.end());
    rep->max_rel_discrepancy = max_rel;
    // flagged list, in (group, signal) order like the reference's loop
    rep->n_flagged = (int64_t)flags.size();
    p->last_flagged.resize(flags.size());
    for (size_t i = 0; i < flags.size(); ++i) {
        tfft_flag& f = p->last_flagged[i];
        f.group = flags[i].first / p->bs;
        f.signal = flags[i].first;
        f.discrepancy = flags[i].second;
        if ((int64_t)i < rep->flagged_cap) rep->flagged[i] = f;
    }
    return TFFT_OK;
}

// Group decisions (protected.py:127-136): more than one flag in a group ->
// unrecoverable, exactly one -> a correction candidate.
void decide(const tfft_plan* p, const std::vector<std::pair<long long, double>>& flags,
            std::vector<int64_t>& bad_groups, std::vector<int64_t>& fix_groups, std::vector<int64_t>& fix_sig) {
    for (size_t i = 0; i < flags.size();) {
        const int64_t g = flags[i].first / p->bs;
        size_t j = i;
        while (j < flags.size() && flags[j].first / p->bs == g) ++j;
        if (j - i > 1) bad_groups.push_back(g);
        else { fix_groups.push_back(g); fix_sig.push_back(flags[i].first); }
        i = j;
    }
}

// Correct the candidate groups of device buffers in/out (groups and signals
// indexed relative to `in`). ONE_SIDED re-transforms the flagged signal from
// the clean input (protected.py:142-147); TWO_SIDED_* rebuilds
// y_f = W s0 - sum_{b != f} y_b and commits only if it re-verifies
// (pipeline.py:164-192). fixed_ok[i] = 1 when group i was corrected.
int correct_groups(tfft_plan* p, const void* in, void* out, int scheme, const void* etw, const void* values,
                   double delta, double abs_floor, int inverse, const std::vector<int64_t>& fix_groups,
                   const std::vector<int64_t>& fix_sig, std::vector<char>& fixed_ok, cudaStream_t st) {
    const int64_t n = p->n;
    int rc;
    fixed_ok.assign(fix_groups.size(), 0);
    if (fix_groups.empty()) return TFFT_OK;
    if (p->single && single_entry(p->prec, p->logn)->fix) {
        // the device correction pass with a host job list (identical
        // arithmetic to the plan-mode pass behind the fused launch)
        const int64_t K = (int64_t)fix_groups.size();
        if (K > p->jobs_cap) {
            cudaFree(p->d_jobs);
            p->d_jobs = nullptr;
            CU(cudaMalloc(&p->d_jobs, K * sizeof(FixJob)));
            p->jobs_cap = K;
        }
        std::vector<FixJob> jobs(K);
        for (int64_t k = 0; k < K; ++k) jobs[k] = FixJob{fix_groups[k] * p->bs, fix_sig[k], 0, 0};
        CU(cudaMemcpyAsync(p->d_jobs, jobs.data(), K * sizeof(FixJob), cudaMemcpyHostToDevice, st));
        rc = launch_fix(p, in, out, etw, values, delta, abs_floor, inverse ? 1 : 0,
                        scheme == TFFT_SCHEME_ONE_SIDED, p->d_jobs, (int)K, st);
        if (rc) return rc;
        CU(cudaMemcpyAsync(jobs.data(), p->d_jobs, K * sizeof(FixJob), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        for (int64_t k = 0; k < K; ++k) fixed_ok[k] = (char)jobs[k].ok;
        return TFFT_OK;
    }
    if (scheme == TFFT_SCHEME_ONE_SIDED) {
        for (size_t i = 0; i < fix_groups.size(); ++i) {
            Launch R = base_launch((const char*)in + fix_sig[i] * n * p->esize,
                                   (char*)out + fix_sig[i] * n * p->esize, 1, inverse ? 1 : 0);
            rc = launch_transform(p, R, st);
            if (rc) return rc;
            fixed_ok[i] = 1;
        }
        return TFFT_OK;
    }
    const int64_t chunk_max = std::max<int64_t>(1, std::min<int64_t>(4096, (int64_t(1) << 28) / (n * (int64_t)p->esize)));
    for (size_t c0 = 0; c0 < fix_groups.size(); c0 += chunk_max) {
        const int64_t K = std::min<int64_t>(chunk_max, fix_groups.size() - c0);
        const long long chunks = (n + FIX_CHUNK - 1) / FIX_CHUNK;
        const size_t tb = p->prec == TFFT_FP32 ? 4 : 8;
        // s0 | W s0 | rebuilt signals | per-chunk checksum partials
        rc = ensure_scratch(p, (size_t)3 * K * n * p->esize + (size_t)K * chunks * 5 * tb);
        if (rc) return rc;
        char* s0 = (char*)p->d_scratch;
        char* ws0 = s0 + (size_t)K * n * p->esize;
        char* fx2 = ws0 + (size_t)K * n * p->esize;
        char* part = fx2 + (size_t)K * n * p->esize;
        if (K > p->jobs_cap) {
            cudaFree(p->d_jobs);
            p->d_jobs = nullptr;
            CU(cudaMalloc(&p->d_jobs, K * sizeof(FixJob)));
            p->jobs_cap = K;
        }
        std::vector<FixJob> jobs(K);
        for (int64_t k = 0; k < K; ++k) {
            jobs[k].first = fix_groups[c0 + k] * p->bs;
            jobs[k].flagged = fix_sig[c0 + k];
            jobs[k].ok = 0;
        }
        CU(cudaMemcpyAsync(p->d_jobs, jobs.data(), K * sizeof(FixJob), cudaMemcpyHostToDevice, st));
        // all K group sums in one launch, then one batched FFT of them
        // one point per thread (the group loop is latency-bound: spread it wide)
        const unsigned gx = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256,
                                                                               (64LL * p->num_sms + K - 1) / K));
        if (p->prec == TFFT_FP32)
            tfft::note_launch(), group_sums_jobs_kernel<float><<<dim3(gx, (unsigned)K), 256, 0, st>>>((const float2*)in, p->bs, n,
                                                                                p->d_jobs, (float2*)s0);
        else
            tfft::note_launch(), group_sums_jobs_kernel<double><<<dim3(gx, (unsigned)K), 256, 0, st>>>((const double2*)in, p->bs, n,
                                                                                 p->d_jobs, (double2*)s0);
        CU(cudaGetLastError());
        Launch W = base_launch(s0, ws0, K, inverse ? 1 : 0);
        rc = launch_transform(p, W, st);
        if (rc) return rc;
        // rebuild + verify + commit, many CTAs per group (the n points in chunks)
        const dim3 g((unsigned)chunks, (unsigned)K);
        if (p->prec == TFFT_FP32) {
            tfft::note_launch(), fix_rebuild_kernel<float><<<g, 256, 0, st>>>((const float2*)in, (const float2*)out, n, p->bs,
                                                        (const float2*)ws0, (float2*)fx2, (const float2*)etw,
                                                        (const float2*)values, p->d_jobs, (float*)part);
            tfft::note_launch(), fix_decide_kernel<float><<<(unsigned)K, 256, 0, st>>>(chunks, (const float*)part, (float)delta,
                                                                (float)abs_floor, 1e-6f, p->d_jobs);
            tfft::note_launch(), fix_commit_kernel<float><<<g, 256, 0, st>>>((float2*)out, n, (const float2*)fx2, p->d_jobs);
        } else {
            tfft::note_launch(), fix_rebuild_kernel<double><<<g, 256, 0, st>>>((const double2*)in, (const double2*)out, n, p->bs,
                                                         (const double2*)ws0, (double2*)fx2, (const double2*)etw,
                                                         (const double2*)values, p->d_jobs, (double*)part);
            tfft::note_launch(), fix_decide_kernel<double><<<(unsigned)K, 256, 0, st>>>(chunks, (const double*)part, delta, abs_floor,
                                                                 1e-12, p->d_jobs);
            tfft::note_launch(), fix_commit_kernel<double><<<g, 256, 0, st>>>((double2*)out, n, (const double2*)fx2, p->d_jobs);
        }
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(jobs.data(), p->d_jobs, K * sizeof(FixJob), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        for (int64_t k = 0; k < K; ++k) fixed_ok[c0 + k] = (char)jobs[k].ok;
    }
    return TFFT_OK;
}

// corrected / unrecoverable lists in group order; recompute accounting
void fill_lists(tfft_plan* p, int scheme, tfft_report* rep, const std::vector<int64_t>& bad_groups,
                const std::vector<int64_t>& fix_groups, const std::vector<int64_t>& fix_sig,
                const std::vector<char>& fixed_ok) {
    if (scheme == TFFT_SCHEME_ONE_SIDED && !fix_groups.empty()) {
        rep->recompute_count = (int64_t)fix_groups.size();
        rep->pass_count += 2 * (int64_t)p->nstages * rep->recompute_count;
    }
    std::vector<int64_t>& unrec = p->last_unrec;
    unrec = bad_groups;
    p->last_corrected.clear();
    for (size_t i = 0; i < fix_groups.size(); ++i) {
        if (fixed_ok[i]) {
            const int64_t nc = (int64_t)p->last_corrected.size();
            if (nc < rep->corrected_cap) {
                rep->corrected_group[nc] = fix_groups[i];
                rep->corrected_signal[nc] = fix_sig[i];
            }
            p->last_corrected.emplace_back(fix_groups[i], fix_sig[i]);
        } else {
            unrec.push_back(fix_groups[i]);
        }
    }
    std::sort(unrec.begin(), unrec.end());
    rep->n_corrected = (int64_t)p->last_corrected.size();
    rep->n_unrecoverable = (int64_t)unrec.size();
    for (size_t i = 0; i < unrec.size() && (int64_t)i < rep->unrecoverable_cap; ++i) rep->unrecoverable[i] = unrec[i];
}

}  // namespace

extern "C" {

int tfft_protect_finish(tfft_plan* p, const void* in, void* out, int64_t batch, int scheme, double delta,
                        double abs_floor, const void* etw, const void* values, int inverse, tfft_report* rep,
                        void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (!rep) return fail(TFFT_EINVAL, "null report");
    if (scheme == TFFT_SCHEME_NONE || batch == 0) return TFFT_OK;
    if (!p->ev_done) return fail(TFFT_EINVAL, "tfft_protect_finish without tfft_protect_launch");
    std::vector<std::pair<long long, double>> flags;
    RecheckFn resolve = [&](const std::vector<long long>& sg, std::vector<double>& rr) {
        return recheck_device(p, in, out, sg, etw, values, abs_floor, rr, st);
    };
    if (p->fix_side) {  // later work on the caller's stream sees the corrected outputs
        CU(cudaStreamWaitEvent(st, p->ev_done, 0));
        p->fix_side = false;
    }
    rc = read_summary(p, batch, st, rep, flags, delta, resolve);  // waits for the summary copy
    if (rc) return rc;
    const FixHead fh = p->h_cnt->fix;
    std::vector<int64_t> bad_groups, fix_groups, fix_sig;
    decide(p, flags, bad_groups, fix_groups, fix_sig);
    std::vector<char> fixed_ok;
    if (fh.ran && !fh.fallback) {
        // corrected on the device already (same grouping, same order)
        if (fh.njobs != (int)fix_groups.size()) return fail(TFFT_ECUDA, "device correction disagrees with the host grouping");
        const FixRes* fr = reinterpret_cast<const FixRes*>(p->h_block + kFixOff);
        fixed_ok.resize(fix_groups.size());
        for (size_t i = 0; i < fix_groups.size(); ++i) {
            if (fr[i].signal != fix_sig[i]) return fail(TFFT_ECUDA, "device correction job mismatch");
            fixed_ok[i] = (char)fr[i].ok;
        }
    } else {
        rc = correct_groups(p, in, out, scheme, etw, values, delta, abs_floor, inverse, fix_groups, fix_sig, fixed_ok,
                            st);
        if (rc) return rc;
    }
    fill_lists(p, scheme, rep, bad_groups, fix_groups, fix_sig, fixed_ok);
    return TFFT_OK;
}

namespace {
struct TileCache {
    std::mutex mu;
    std::map<std::pair<int64_t, int>, tfft_plan*> plans;
    void* d_buf = nullptr;
    size_t d_bytes = 0;
};
TileCache g_tile;
}  // namespace

int tfft_tile_fft(const void* in, void* out, int64_t t, int64_t l, int dtype_bytes, int inverse, int host,
                  void* stream) {
    if (dtype_bytes != 8 && dtype_bytes != 16) return fail(TFFT_EINVAL, "unsupported dtype");
    if (t < 0 || l < 1 || !is_pow2(l)) return fail(TFFT_EINVAL, "tiles must be (T, L) with L a power of two");
    if (t == 0) return TFFT_OK;
    if (!in || !out) return fail(TFFT_EINVAL, "null buffer");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bytes = (size_t)t * l * dtype_bytes;
    if (l == 1) {
        CU(cudaMemcpyAsync(out, in, bytes, host ? cudaMemcpyHostToHost : cudaMemcpyDeviceToDevice, st));
        if (host) CU(cudaStreamSynchronize(st));
        return TFFT_OK;
    }
    std::lock_guard<std::mutex> lk(g_tile.mu);
    const int prec = dtype_bytes == 8 ? TFFT_FP32 : TFFT_FP64;
    auto key = std::make_pair(l, prec);
    tfft_plan* p;
    auto it = g_tile.plans.find(key);
    if (it == g_tile.plans.end()) {
        const int e = ilog2(l);
        const int cnt = l <= (1 << 13) ? 1 : (l <= (1 << 22) ? 2 : 3);
        int64_t dims[3];
        const int base = e / cnt, rem = e % cnt;
        for (int i = 0; i < cnt; ++i) dims[i] = int64_t(1) << (base + (i >= cnt - rem ? 1 : 0));
        int device = 0;
        CU(cudaGetDevice(&device));
        int rc = tfft_plan_create(&p, l, prec, cnt, dims, 1, device);
        if (rc) return rc;
        g_tile.plans[key] = p;
    } else {
        p = it->second;
    }
    const void* din = in;
    void* dout = out;
    if (host) {
        if (2 * bytes > g_tile.d_bytes) {
            cudaFree(g_tile.d_buf);
            g_tile.d_buf = nullptr;
            g_tile.d_bytes = 0;
            CU(cudaMalloc(&g_tile.d_buf, 2 * bytes));
            g_tile.d_bytes = 2 * bytes;
        }
        CU(cudaMemcpyAsync(g_tile.d_buf, in, bytes, cudaMemcpyHostToDevice, st));
        din = g_tile.d_buf;
        dout = (char*)g_tile.d_buf + bytes;
    }
    Launch L = base_launch(din, dout, t, inverse ? 1 : 0);
    L.scale_inv = 0;  // tile_fft leaves scaling to the caller (_stockham.pyx:46-65)
    int rc = launch_transform(p, L, st);
    if (rc) return rc;
    if (host) {
        CU(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    return TFFT_OK;
}

// Host-buffer drop-in of run_protected (the numpy path of the reference,
// protected.py:63-166): the batch streams through a ring of device chunks —
// H2D of chunk i+1, the fused protected transform of chunk i and D2H of chunk
// i-1 run concurrently on three streams. Chunks are whole checksum groups and
// keep their global signal indices (sig_base), so flags, the fault and the
// report are those of one call over the whole batch. Flagged groups (rare)
// are re-staged afterwards and corrected on the device like the device path.
int tfft_run_protected_host(tfft_plan* p, const void* in, void* out, int64_t batch, int scheme, double delta,
                            double abs_floor, const void* etw, const void* values, const tfft_fault* fault,
                            int inverse, tfft_report* rep, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Launch L;
    rc = prepare_protected(p, in, out, batch, scheme, delta, etw, values, abs_floor, fault, inverse, rep, L);
    if (rc) return rc;
    if (batch == 0) return TFFT_OK;
    const bool prot = scheme != TFFT_SCHEME_NONE;
    const size_t sig_bytes = (size_t)p->n * p->esize;
    const size_t grp_bytes = sig_bytes * p->bs;
    const int64_t gpc = groups_per_chunk(p, batch);
    const size_t chunk = (size_t)gpc * grp_bytes;
    rc = ensure_ring(p, chunk, st);
    if (rc) return rc;
    if (prot) {
        rc = ensure_flags(p, batch);
        if (rc) return rc;
        CU(cudaMemsetAsync(p->d_cnt, 0, sizeof(Counters), st));
    }
    // the copy streams start behind whatever the caller queued on `st`
    CU(cudaEventRecord(p->ev_done, st));
    CU(cudaStreamWaitEvent(p->s_h2d, p->ev_done, 0));
    CU(cudaStreamWaitEvent(p->s_d2h, p->ev_done, 0));
    const int64_t spc = gpc * p->bs;  // signals per chunk
    const int64_t nchunks = (batch + spc - 1) / spc;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int slot = (int)(c % tfft_plan::kRing);
        char* din = (char*)p->ring + (size_t)slot * 2 * p->ring_chunk;
        char* dout = din + p->ring_chunk;
        const int64_t s0 = c * spc;
        const int64_t ns = std::min<int64_t>(spc, batch - s0);
        const size_t bytes = (size_t)ns * sig_bytes;
        if (c >= tfft_plan::kRing) {  // slot reuse: its last transform and D2H are done
            CU(cudaStreamWaitEvent(p->s_h2d, p->ev_comp[slot], 0));
        }
        CU(cudaMemcpyAsync(din, (const char*)in + s0 * sig_bytes, bytes, cudaMemcpyHostToDevice, p->s_h2d));
        CU(cudaEventRecord(p->ev_in[slot], p->s_h2d));
        CU(cudaStreamWaitEvent(st, p->ev_in[slot], 0));
        if (c >= tfft_plan::kRing) CU(cudaStreamWaitEvent(st, p->ev_out[slot], 0));
        Launch C = L;
        C.in = din;
        C.out = dout;
        C.batch = ns;
        C.sig_base = s0;
        rc = launch_transform(p, C, st);
        if (rc) return rc;
        CU(cudaEventRecord(p->ev_comp[slot], st));
        CU(cudaStreamWaitEvent(p->s_d2h, p->ev_comp[slot], 0));
        CU(cudaMemcpyAsync((char*)out + s0 * sig_bytes, dout, bytes, cudaMemcpyDeviceToHost, p->s_d2h));
        CU(cudaEventRecord(p->ev_out[slot], p->s_d2h));
    }
    // join: `st` waits for the last D2H so callers may sync on their stream
    CU(cudaEventRecord(p->ev_out[0], p->s_d2h));
    CU(cudaStreamWaitEvent(st, p->ev_out[0], 0));
    if (!prot) return cudaStreamSynchronize(st) == cudaSuccess ? TFFT_OK : fail(TFFT_ECUDA, "stream sync");
    rc = enqueue_summary(p, st);
    if (rc) return rc;
    CU(cudaStreamSynchronize(st));
    std::vector<std::pair<long long, double>> flags;
    RecheckFn resolve = [&](const std::vector<long long>& sg, std::vector<double>& rr) {
        // rare: stage the signals' input and output rows
        StageFn stage = [&](int64_t first, int64_t cnt, char* di, char* dq) {
            CU(cudaMemcpyAsync(di, (const char*)in + first * sig_bytes, cnt * sig_bytes, cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(dq, (const char*)out + first * sig_bytes, cnt * sig_bytes, cudaMemcpyHostToDevice,
                               st));
            return (int)TFFT_OK;
        };
        return recheck_staged(p, sg, rr, etw, values, abs_floor, stage, st);
    };
    rc = read_summary(p, batch, st, rep, flags, delta, resolve);
    if (rc) return rc;
    std::vector<int64_t> bad_groups, fix_groups, fix_sig;
    decide(p, flags, bad_groups, fix_groups, fix_sig);
    std::vector<char> fixed_ok(fix_groups.size(), 0);
    // rare path: re-stage each candidate group (clean input + current output)
    // into ring slot 0 and correct it there
    char* din = (char*)p->ring;
    char* dout = din + p->ring_chunk;
    for (size_t i = 0; i < fix_groups.size(); ++i) {
        const int64_t g = fix_groups[i];
        const size_t off = (size_t)g * grp_bytes;
        CU(cudaMemcpyAsync(din, (const char*)in + off, grp_bytes, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(dout, (const char*)out + off, grp_bytes, cudaMemcpyHostToDevice, st));
        std::vector<int64_t> g1{0}, s1{fix_sig[i] - g * p->bs};
        std::vector<char> ok1;
        rc = correct_groups(p, din, dout, scheme, etw, values, delta, abs_floor, inverse, g1, s1, ok1, st);
        if (rc) return rc;
        if (ok1[0]) CU(cudaMemcpyAsync((char*)out + off, dout, grp_bytes, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        fixed_ok[i] = ok1[0];
    }
    fill_lists(p, scheme, rep, bad_groups, fix_groups, fix_sig, fixed_ok);
    return TFFT_OK;
}

// Batched fault campaign (reference fault_lab/campaign.py:95-195): `runs`
// independent protected calls of `run_batch` signals fused into one launch,
// each run with its own single fault (faults[r], run-relative signal).
int tfft_run_campaign(tfft_plan* p, const void* in, void* out, int64_t runs, int64_t run_batch, int scheme,
                      double delta, double abs_floor, const void* etw, const void* values,
                      const tfft_fault* faults, int inverse, double* run_max_rel, int32_t* run_fired,
                      tfft_report* rep, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (runs < 1 || run_batch < 1) return fail(TFFT_EINVAL, "runs and run_batch must be >= 1");
    if (run_batch % p->bs) return fail(TFFT_EINVAL, "run_batch not divisible by group size");
    if (scheme == TFFT_SCHEME_NONE) return fail(TFFT_EINVAL, "a campaign needs a protected scheme");
    if (!run_max_rel) return fail(TFFT_EINVAL, "null run_max_rel");
    const int64_t batch = runs * run_batch;
    Launch L;
    rc = prepare_protected(p, in, out, batch, scheme, delta, etw, values, abs_floor, nullptr, inverse, rep, L);
    if (rc) return rc;
    // ---- per-run faults, translated like the single-fault path
    std::vector<FaultRec> tab;
    std::vector<HostFault> hf;
    bool any = false;
    if (faults) {
        if (p->single) tab.assign(runs, FaultRec{});
        else hf.assign(runs, HostFault{});
        for (int64_t r = 0; r < runs; ++r) {
            FaultT ft;
            rc = translate_fault(p, faults[r], run_batch, ft);
            if (rc) return rc;
            if (run_fired) run_fired[r] = ft.where != AT_NONE;
            if (ft.where == AT_NONE) continue;
            any = true;
            if (p->single) {
                tab[r].pos = ft.elem;
                tab[r].signal = (int)ft.signal;
                tab[r].where = ft.where;
                tab[r].comp = ft.comp;
                tab[r].bit = ft.bit;
            } else {
                hf[r].signal = ft.signal;
                hf[r].elem = ft.elem;
                hf[r].where = ft.where;
                hf[r].stage = ft.stage;
                hf[r].comp = ft.comp;
                hf[r].bit = ft.bit;
            }
        }
    } else if (run_fired) {
        for (int64_t r = 0; r < runs; ++r) run_fired[r] = 0;
    }
    if (any) {
        L.f_div = run_batch;
        if (p->single) {
            const size_t bytes = tab.size() * sizeof(FaultRec);
            if (bytes > p->ftab_bytes) {
                cudaFree(p->d_ftab);
                p->d_ftab = nullptr;
                p->ftab_bytes = 0;
                CU(cudaMalloc(&p->d_ftab, bytes));
                p->ftab_bytes = bytes;
            }
            CU(cudaMemcpyAsync(p->d_ftab, tab.data(), bytes, cudaMemcpyHostToDevice, st));
            L.f_table = (const FaultRec*)p->d_ftab;
        } else {
            L.faults = hf.data();
            L.nfaults = runs;
        }
    }
    const size_t tb = p->prec == TFFT_FP32 ? 4 : 8;
    if (batch * tb > p->rel_bytes) {
        cudaFree(p->d_rel);
        p->d_rel = nullptr;
        p->rel_bytes = 0;
        CU(cudaMalloc(&p->d_rel, batch * tb));
        p->rel_bytes = batch * tb;
    }
    L.rel_out = p->d_rel;
    rc = ensure_flags(p, batch);
    if (rc) return rc;
    CU(cudaMemsetAsync(p->d_cnt, 0, sizeof(Counters), st));
    rc = launch_transform(p, L, st);
    if (rc) return rc;
    rc = enqueue_summary(p, st);
    if (rc) return rc;
    std::vector<std::pair<long long, double>> flags;
    std::vector<std::pair<long long, double>> rechecked;
    RecheckFn resolve = [&](const std::vector<long long>& sg, std::vector<double>& rr) {
        return recheck_device(p, in, out, sg, etw, values, abs_floor, rr, st);
    };
    rc = read_summary(p, batch, st, rep, flags, delta, resolve, &rechecked);
    if (rc) return rc;
    // per-run max discrepancy (protected.py:124-126 max over the run's groups)
    std::vector<char> rel((size_t)batch * tb);
    CU(cudaMemcpyAsync(rel.data(), p->d_rel, batch * tb, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (const auto& rc_ : rechecked) {  // exact values of the recheck sentinels
        if (tb == 4) ((float*)rel.data())[rc_.first] = (float)rc_.second;
        else ((double*)rel.data())[rc_.first] = rc_.second;
    }
    for (int64_t r = 0; r < runs; ++r) {
        double mx = 0.0;
        for (int64_t i = r * run_batch; i < (r + 1) * run_batch; ++i) {
            const double v = tb == 4 ? (double)((const float*)rel.data())[i] : ((const double*)rel.data())[i];
            if (v > mx || v != v) mx = v != v ? INFINITY : v;
        }
        run_max_rel[r] = mx;
    }
    std::vector<int64_t> bad_groups, fix_groups, fix_sig;
    decide(p, flags, bad_groups, fix_groups, fix_sig);
    std::vector<char> fixed_ok;
    rc = correct_groups(p, in, out, scheme, etw, values, delta, abs_floor, inverse, fix_groups, fix_sig, fixed_ok, st);
    if (rc) return rc;
    fill_lists(p, scheme, rep, bad_groups, fix_groups, fix_sig, fixed_ok);
    rep->fault_fired = any;
    return TFFT_OK;
}

}  // extern "C"

namespace {

struct Fd {
    int fd = -1;
    ~Fd() { if (fd >= 0) close(fd); }
};

int io_fail(const char* what, const char* path) {
    return fail(TFFT_EIO, std::string(what) + " " + path + ": " + strerror(errno));
}

// full-length pread / pwrite (short transfers retried)
bool read_at(int fd, void* buf, size_t bytes, off_t off) {
    char* b = (char*)buf;
    while (bytes) {
        const ssize_t r = pread(fd, b, bytes, off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) return false;
        b += r; off += r; bytes -= (size_t)r;
    }
    return true;
}
// Temp output of an in-place file transform: renamed over `target` by
// commit(), removed if the call fails before that.
struct TempOut {
    std::string path, target;
    int commit() {
        if (path.empty()) return TFFT_OK;
        if (rename(path.c_str(), target.c_str()) != 0) return io_fail("cannot replace", target.c_str());
        path.clear();
        return TFFT_OK;
    }
    ~TempOut() {
        if (!path.empty()) unlink(path.c_str());
    }
};

bool write_at(int fd, const void* buf, size_t bytes, off_t off) {
    const char* b = (const char*)buf;
    while (bytes) {
        const ssize_t r = pwrite(fd, b, bytes, off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) return false;
        b += r; off += r; bytes -= (size_t)r;
    }
    return true;
}

}  // namespace

extern "C" {

int tfft_signal_file_batch(const char* path, int64_t n, int precision, int64_t* batch) {
    if (!path || !batch) return fail(TFFT_EINVAL, "null argument");
    if (precision != TFFT_FP32 && precision != TFFT_FP64) return fail(TFFT_EINVAL, "bad precision");
    struct stat sb;
    if (stat(path, &sb) != 0) return io_fail("cannot stat", path);
    const int64_t sig = n * (precision == TFFT_FP32 ? 8 : 16);
    if (sb.st_size == 0 || sb.st_size % sig) {
        return fail(TFFT_EINVAL, "input length mismatch: " + std::to_string((long long)sb.st_size) +
                                     " bytes is not a whole number of " + std::to_string((long long)n) +
                                     "-sample " + (precision == TFFT_FP32 ? "fp32" : "fp64") + " signals");
    }
    *batch = sb.st_size / sig;
    return TFFT_OK;
}

// cli.py:54-67 cmd_transform + signal_io.py:11-33: raw interleaved (re, im)
// little-endian files are the complex64 / complex128 memory layout, so the
// file is streamed chunk by chunk: pread into a pinned slot -> H2D -> fused
// protected transform -> D2H into a pinned slot -> pwrite by a writer thread,
// all stages of different chunks in flight at once.
int tfft_run_protected_file(tfft_plan* p, const char* in_path, const char* out_path, int scheme, double delta,
                            double abs_floor, const void* etw, const void* values, const tfft_fault* fault,
                            int inverse, int64_t* batch_out, tfft_report* rep, void* stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    if (!in_path || !out_path) return fail(TFFT_EINVAL, "null path");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t batch = 0;
    rc = tfft_signal_file_batch(in_path, p->n, p->prec, &batch);
    if (rc) return rc;
    if (batch_out) *batch_out = batch;
    Launch L;
    static char dummy;
    rc = prepare_protected(p, &dummy, &dummy, batch, scheme, delta, etw, values, abs_floor, fault, inverse, rep, L);
    if (rc) return rc;
    const bool prot = scheme != TFFT_SCHEME_NONE;
    Fd fin, fout;
    fin.fd = open(in_path, O_RDONLY);
    if (fin.fd < 0) return io_fail("cannot open", in_path);
    // Output == input (the same file, or a link to it): the reference reads
    // the whole input before it writes (cli.py:54-67), so the result streams
    // into a temp file next to the target and is renamed over it at the end;
    // the input stays intact until then (also on failure: the temp is removed).
    TempOut tmp;
    std::string wpath = out_path;
    {
        struct stat si, so;
        if (fstat(fin.fd, &si) == 0 && stat(out_path, &so) == 0 && si.st_dev == so.st_dev && si.st_ino == so.st_ino) {
            char* real = realpath(out_path, nullptr);
            if (!real) return io_fail("cannot resolve", out_path);
            tmp.target = real;
            free(real);
            std::string t = tmp.target + ".tfft-XXXXXX";
            std::vector<char> tmpl(t.begin(), t.end());
            tmpl.push_back(0);
            fout.fd = mkstemp(tmpl.data());
            if (fout.fd < 0) return io_fail("cannot create a temp file for", out_path);
            tmp.path = tmpl.data();
            if (fchmod(fout.fd, so.st_mode & 07777) != 0) return io_fail("cannot chmod", tmp.path.c_str());
            wpath = tmp.path;
        }
    }
    if (tmp.path.empty()) {
        fout.fd = open(out_path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (fout.fd < 0) return io_fail("cannot create", out_path);
    }
    const size_t sig_bytes = (size_t)p->n * p->esize;
    const size_t grp_bytes = sig_bytes * p->bs;
    if (ftruncate(fout.fd, (off_t)(batch * sig_bytes)) != 0) return io_fail("cannot size", out_path);
    const int64_t gpc = groups_per_chunk(p, batch);
    const size_t chunk = (size_t)gpc * grp_bytes;
    rc = ensure_ring(p, chunk, st);
    if (rc) return rc;
    constexpr int R = tfft_plan::kRing;
    if (chunk > p->h_stage_chunk) {
        if (p->h_stage) cudaFreeHost(p->h_stage);
        p->h_stage = nullptr;
        p->h_stage_chunk = 0;
        if (cudaHostAlloc(&p->h_stage, 2 * R * chunk, cudaHostAllocDefault) != cudaSuccess)
            return fail(TFFT_ENOMEM, "pinned file staging");
        p->h_stage_chunk = chunk;
    }
    auto hin = [&](int slot) { return (char*)p->h_stage + (size_t)slot * 2 * p->h_stage_chunk; };
    auto hout = [&](int slot) { return hin(slot) + p->h_stage_chunk; };
    if (prot) {
        rc = ensure_flags(p, batch);
        if (rc) return rc;
        CU(cudaMemsetAsync(p->d_cnt, 0, sizeof(Counters), st));
    }
    CU(cudaEventRecord(p->ev_done, st));
    CU(cudaStreamWaitEvent(p->s_h2d, p->ev_done, 0));
    CU(cudaStreamWaitEvent(p->s_d2h, p->ev_done, 0));
    const int64_t spc = gpc * p->bs;
    const int64_t nchunks = (batch + spc - 1) / spc;

    // writer: retires chunks in order (waits for their D2H, pwrites them)
    std::mutex mu;
    std::condition_variable cv;
    int64_t queued = 0, written = 0;  // chunks handed to / finished by the writer
    std::atomic<int> werr{0};
    std::string werr_msg;
    std::thread writer([&] {
        for (int64_t c = 0; c < nchunks; ++c) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return queued > c || werr.load(); });
            }
            if (werr.load()) break;
            const int slot = (int)(c % R);
            const int64_t s0 = c * spc;
            const size_t bytes = (size_t)std::min<int64_t>(spc, batch - s0) * sig_bytes;
            if (cudaEventSynchronize(p->ev_out[slot]) != cudaSuccess) {
                werr_msg = "D2H failed";
                werr = TFFT_ECUDA;
            } else if (!write_at(fout.fd, hout(slot), bytes, (off_t)(s0 * sig_bytes))) {
                werr_msg = std::string("cannot write ") + out_path + ": " + strerror(errno);
                werr = TFFT_EIO;
            }
            {
                std::lock_guard<std::mutex> lk(mu);
                written = c + 1;
            }
            cv.notify_all();
            if (werr.load()) break;
        }
    });
    auto stop_writer = [&](int code, const std::string& msg) {
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!werr.load()) {
                werr = code ? code : TFFT_ECUDA;
                werr_msg = msg;
            }
        }
        cv.notify_all();
        writer.join();
        return fail(werr.load(), werr_msg);
    };
    for (int64_t c = 0; c < nchunks; ++c) {
        const int slot = (int)(c % R);
        char* din = (char*)p->ring + (size_t)slot * 2 * p->ring_chunk;
        char* dout = din + p->ring_chunk;
        const int64_t s0 = c * spc;
        const int64_t ns = std::min<int64_t>(spc, batch - s0);
        const size_t bytes = (size_t)ns * sig_bytes;
        {  // slot free: the writer has retired chunk c - R
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return written >= c - R + 1 || werr.load(); });
        }
        if (werr.load()) {
            writer.join();
            return fail(werr.load(), werr_msg);
        }
        if (!read_at(fin.fd, hin(slot), bytes, (off_t)(s0 * sig_bytes)))
            return stop_writer(TFFT_EIO, std::string("cannot read ") + in_path + ": " + strerror(errno));
        if (cudaMemcpyAsync(din, hin(slot), bytes, cudaMemcpyHostToDevice, p->s_h2d) != cudaSuccess ||
            cudaEventRecord(p->ev_in[slot], p->s_h2d) != cudaSuccess ||
            cudaStreamWaitEvent(st, p->ev_in[slot], 0) != cudaSuccess)
            return stop_writer(TFFT_ECUDA, "H2D enqueue failed");
        Launch C = L;
        C.in = din;
        C.out = dout;
        C.batch = ns;
        C.sig_base = s0;
        rc = launch_transform(p, C, st);
        if (rc) return stop_writer(rc, g_err);
        if (cudaEventRecord(p->ev_comp[slot], st) != cudaSuccess ||
            cudaStreamWaitEvent(p->s_d2h, p->ev_comp[slot], 0) != cudaSuccess ||
            cudaMemcpyAsync(hout(slot), dout, bytes, cudaMemcpyDeviceToHost, p->s_d2h) != cudaSuccess ||
            cudaEventRecord(p->ev_out[slot], p->s_d2h) != cudaSuccess)
            return stop_writer(TFFT_ECUDA, "D2H enqueue failed");
        {
            std::lock_guard<std::mutex> lk(mu);
            queued = c + 1;
        }
        cv.notify_all();
    }
    writer.join();
    if (werr.load()) return fail(werr.load(), werr_msg);
    CU(cudaStreamSynchronize(p->s_d2h));
    if (!prot) return tmp.commit();
    rc = enqueue_summary(p, st);
    if (rc) return rc;
    std::vector<std::pair<long long, double>> flags;
    RecheckFn resolve = [&](const std::vector<long long>& sg, std::vector<double>& rr) {
        Fd fo;
        fo.fd = open(wpath.c_str(), O_RDONLY);
        if (fo.fd < 0) return io_fail("cannot reopen", wpath.c_str());
        // rare: re-stage the signals' rows from the files
        StageFn stage = [&](int64_t first, int64_t cnt, char* di, char* dq) {
            const off_t off = (off_t)(first * sig_bytes);
            const size_t bytes = (size_t)cnt * sig_bytes;
            CU(cudaStreamSynchronize(st));  // the pinned slot is reused per run
            if (!read_at(fin.fd, hin(0), bytes, off)) return io_fail("cannot read", in_path);
            if (!read_at(fo.fd, hout(0), bytes, off)) return io_fail("cannot read", wpath.c_str());
            CU(cudaMemcpyAsync(di, hin(0), bytes, cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(dq, hout(0), bytes, cudaMemcpyHostToDevice, st));
            return (int)TFFT_OK;
        };
        return recheck_staged(p, sg, rr, etw, values, abs_floor, stage, st);
    };
    rc = read_summary(p, batch, st, rep, flags, delta, resolve);
    if (rc) return rc;
    std::vector<int64_t> bad_groups, fix_groups, fix_sig;
    decide(p, flags, bad_groups, fix_groups, fix_sig);
    std::vector<char> fixed_ok(fix_groups.size(), 0);
    // rare path: each candidate group's clean input and current output are
    // re-staged from the files, corrected on the device and written back
    char* din = (char*)p->ring;
    char* dout = din + p->ring_chunk;
    int infd2 = open(wpath.c_str(), O_RDONLY);
    if (!fix_groups.empty() && infd2 < 0) return io_fail("cannot reopen", wpath.c_str());
    Fd fo2;
    fo2.fd = infd2;
    for (size_t i = 0; i < fix_groups.size(); ++i) {
        const int64_t g = fix_groups[i];
        const off_t off = (off_t)(g * grp_bytes);
        if (!read_at(fin.fd, hin(0), grp_bytes, off)) return io_fail("cannot read", in_path);
        if (!read_at(fo2.fd, hout(0), grp_bytes, off)) return io_fail("cannot read", wpath.c_str());
        CU(cudaMemcpyAsync(din, hin(0), grp_bytes, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(dout, hout(0), grp_bytes, cudaMemcpyHostToDevice, st));
        std::vector<int64_t> g1{0}, s1{fix_sig[i] - g * p->bs};
        std::vector<char> ok1;
        rc = correct_groups(p, din, dout, scheme, etw, values, delta, abs_floor, inverse, g1, s1, ok1, st);
        if (rc) return rc;
        if (ok1[0]) {
            CU(cudaMemcpyAsync(hout(0), dout, grp_bytes, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            if (!write_at(fout.fd, hout(0), grp_bytes, off)) return io_fail("cannot write", out_path);
        }
        fixed_ok[i] = ok1[0];
    }
    fill_lists(p, scheme, rep, bad_groups, fix_groups, fix_sig, fixed_ok);
    return tmp.commit();
}

}  // extern "C"

extern "C" {

int tfft_element_encode(int r, int64_t B, const void* x, void* y, const void* etw_row, const void* vals_col,
                        void* row_in, void* xe, void* stream) {
    if (r < 1 || r > 32 || B < 1) return fail(TFFT_EINVAL, "tile must be r x B with 1 <= r <= 32");
    if (!x || !y || !etw_row || !vals_col || !row_in || !xe) return fail(TFFT_EINVAL, "null buffer");
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = (int)std::min<long long>((B + 127) / 128, 1024);
    tfft::note_launch(), element_encode_kernel<<<std::max(grid, 1), 128, 0, st>>>(r, B, (const double2*)x, (const double2*)etw_row,
                                                               (const double2*)vals_col, (double2*)y,
                                                               (double2*)row_in, (double2*)xe);
    CU(cudaGetLastError());
    return TFFT_OK;
}

int tfft_element_verify(int r, int64_t B, void* y, const void* row_in, const void* xe, const void* vals_row,
                        const void* vals_col, double delta, double abs_floor, void* rel, int32_t* result,
                        void* stream) {
    if (r < 1 || r > 32 || B < 1) return fail(TFFT_EINVAL, "tile must be r x B with 1 <= r <= 32");
    if (!y || !row_in || !xe || !vals_row || !vals_col || !rel || !result) return fail(TFFT_EINVAL, "null buffer");
    cudaStream_t st = (cudaStream_t)stream;
    int* d_res = nullptr;
    CU(cudaMallocAsync((void**)&d_res, 3 * sizeof(int), st));
    CU(cudaMemsetAsync(d_res, 0, 3 * sizeof(int), st));
    tfft::note_launch(), element_verify_kernel<<<1, AUX_THREADS, 0, st>>>(r, B, (double2*)y, (const double2*)row_in, (const double2*)xe,
                                                     (const double2*)vals_row, (const double2*)vals_col, delta,
                                                     abs_floor, (double*)rel, d_res);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(result, d_res, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaFreeAsync(d_res, st));
    CU(cudaStreamSynchronize(st));
    return TFFT_OK;
}

}  // extern "C"

extern "C" {

int tfft_set_device_correction(tfft_plan* p, int enable) {
    if (!p) return fail(TFFT_EINVAL, "null plan");
    p->dev_fix = enable ? 1 : 0;
    return TFFT_OK;
}

int tfft_set_check_level(tfft_plan* p, int level) {
    if (!p) return fail(TFFT_EINVAL, "null plan");
    if (level != 0 && level != 1) return fail(TFFT_EINVAL, "check level must be 0 (threadblock) or 1 (thread)");
    if (level == 1 && !p->single) return fail(TFFT_EUNSUPPORTED, "thread-level checks are built for n <= 2^13");
    p->check_level = level;
    return TFFT_OK;
}

}  // extern "C"

extern "C" {

int tfft_dft(const void* in, void* out, int64_t batch, int64_t n, int inverse, void* stream) {
    if (n < 1 || batch < 0) return fail(TFFT_EINVAL, "bad shape");
    if (n > (int64_t(1) << 14)) return fail(TFFT_EINVAL, "oracle limited to n <= 16384");
    if (batch == 0) return TFFT_OK;
    if (!in || !out) return fail(TFFT_EINVAL, "null buffer");
    cudaStream_t st = (cudaStream_t)stream;
    // w^m = exp(-+ 2 pi i m / n), m < n, rounded once from long double
    std::vector<double2> w(n);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int64_t m = 0; m < n; ++m) {
        const long double a = two_pi * (long double)m / (long double)n;
        w[m] = make_double2((double)cosl(a), (double)((inverse ? 1.0L : -1.0L) * sinl(a)));
    }
    double2* dw = nullptr;
    CU(cudaMallocAsync((void**)&dw, n * sizeof(double2), st));
    CU(cudaMemcpyAsync(dw, w.data(), n * sizeof(double2), cudaMemcpyHostToDevice, st));
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int64_t nb = std::min<int64_t>(65535, batch - b0);
        tfft::note_launch(), dft_direct_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)nb), 256, 0, st>>>(
            (const double2*)in + b0 * n, (double2*)out + b0 * n, n, dw, inverse ? 1.0 / (double)n : 1.0);
        CU(cudaGetLastError());
    }
    CU(cudaFreeAsync(dw, st));
    CU(cudaStreamSynchronize(st));  // the host table lives on this frame
    return TFFT_OK;
}

int tfft_launch_count(int64_t* count) {
    if (!count) return fail(TFFT_EINVAL, "null argument");
    *count = tfft::g_launches.load();
    return TFFT_OK;
}

int tfft_report_fetch(const tfft_plan* p, tfft_report* rep) {
    if (!p || !rep) return fail(TFFT_EINVAL, "null argument");
    rep->n_flagged = (int64_t)p->last_flagged.size();
    rep->n_corrected = (int64_t)p->last_corrected.size();
    rep->n_unrecoverable = (int64_t)p->last_unrec.size();
    for (int64_t i = 0; i < rep->n_flagged && i < rep->flagged_cap; ++i) rep->flagged[i] = p->last_flagged[i];
    for (int64_t i = 0; i < rep->n_corrected && i < rep->corrected_cap; ++i) {
        rep->corrected_group[i] = p->last_corrected[i].first;
        rep->corrected_signal[i] = p->last_corrected[i].second;
    }
    for (int64_t i = 0; i < rep->n_unrecoverable && i < rep->unrecoverable_cap; ++i)
        rep->unrecoverable[i] = p->last_unrec[i];
    return TFFT_OK;
}

int tfft_plan_exec_passes(const tfft_plan* p) {
    if (!p) return -1;
    if (p->single) return 1;
    return p->have_fast ? 3 : p->nstages;
}

}  // extern "C"
