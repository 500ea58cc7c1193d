// Host side of the multi-launch path: twiddle tables, workspace and the
// per-stage launch sequence (reference fft_core/execute.py:82-106 — each
// reference stage is one launch here; the transposes become address maps).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tfft.h"
#include "multi.cuh"
#include "registry.h"

namespace tfft {

namespace {
thread_local std::string m_err;
int merr(int code, const std::string& s) {
    m_err = s;
    return code;
}
#define MCU(call)                                                                            \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return merr(TFFT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int lg(long long n) {
    int l = 0;
    while ((1ll << l) < n) ++l;
    return l;
}

// exp(-2 pi i k / N) with quadrant symmetry (long double).
void root(long long N, long long k, long double* re, long double* im) {
    k %= N;
    if (k < 0) k += N;
    const long double two_pi = 6.283185307179586476925286766559005768L;
    long double c, s;
    if ((4 * k) % N == 0) {
        const int q = (int)((4 * k) / N);
        c = q == 0 ? 1.0L : (q == 2 ? -1.0L : 0.0L);
        s = q == 1 ? 1.0L : (q == 3 ? -1.0L : 0.0L);
    } else {
        const long long qn = N / 4;
        const int q = (int)(k / qn);
        const long long r = k - q * qn;
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

int upload_roots(int prec, long long N, long long count, long long stride, void** dst) {
    const size_t es = prec == TFFT_FP32 ? 8 : 16;
    MCU(cudaMalloc(dst, count * es));
    std::vector<unsigned char> h(count * es);
    for (long long k = 0; k < count; ++k) {
        long double re, im;
        root(N, k * stride, &re, &im);
        if (prec == TFFT_FP32) {
            float2 v = make_float2((float)re, (float)im);
            memcpy(&h[k * es], &v, es);
        } else {
            double2 v = make_double2((double)re, (double)im);
            memcpy(&h[k * es], &v, es);
        }
    }
    MCU(cudaMemcpy(*dst, h.data(), count * es, cudaMemcpyHostToDevice));
    return TFFT_OK;
}

// t[M + k] = w_M^k for all powers of two M <= L (the engine's pass twiddles)
int upload_multires(int prec, long long L, void** dst) {
    const size_t es = prec == TFFT_FP32 ? 8 : 16;
    MCU(cudaMalloc(dst, 2 * L * es));
    std::vector<unsigned char> h(2 * L * es, 0);
    for (long long M = 1; M <= L; M *= 2) {
        for (long long k = 0; k < M; ++k) {
            long double re = 1.0L, im = 0.0L;
            if (M >= 2) root(M, k, &re, &im);
            if (prec == TFFT_FP32) {
                float2 v = make_float2((float)re, (float)im);
                memcpy(&h[(M + k) * es], &v, es);
            } else {
                double2 v = make_double2((double)re, (double)im);
                memcpy(&h[(M + k) * es], &v, es);
            }
        }
    }
    MCU(cudaMemcpy(*dst, h.data(), 2 * L * es, cudaMemcpyHostToDevice));
    return TFFT_OK;
}

int g_pass_override[2][12][3] = {};  // variant + 1; 0 = tuned choice

const PassEntry* pass_variant(int prec, int logl, int variant) {
    const PassEntry* tab = prec == TFFT_FP32 ? kPass_fp32 : kPass_fp64;
    const int cnt = prec == TFFT_FP32 ? kPassCount_fp32 : kPassCount_fp64;
    for (int i = 0; i < cnt; ++i)
        if (tab[i].logl == logl && tab[i].variant == variant) return &tab[i];
    return nullptr;
}

// the entry stage kind `kind` of dim 2^logl launches
const PassEntry* pass_entry(int prec, int logl, int kind) {
    if (logl < 0 || logl >= 12) return nullptr;
    const int ov = g_pass_override[prec][logl][kind];
    const int v = ov > 0 ? ov - 1 : (prec == TFFT_FP32 ? kPassChoice_fp32 : kPassChoice_fp64)[logl][kind];
    const PassEntry* e = pass_variant(prec, logl, v);
    return e ? e : pass_variant(prec, logl, 0);
}

int kind_of(int k, int nst) { return k == 0 ? KIND_FIRST : (k == nst - 1 ? KIND_LAST : KIND_MID); }

// A fault (where 1 input / 2 stage:`stage` / 3 output, element e in the
// reference layout of that hook) in pass k's tile coordinates; returns the
// pass's where code (0: not in this pass).
int pass_fault(int k, int nst, long long d0, long long d1, long long d2, long long R0, int where, int stage,
               long long e, long long& unit, int& idx) {
    const int kind = kind_of(k, nst);
    if (where == 1 && k == 0) {                 // input: x[j*R0 + c]
        unit = e % R0; idx = (int)(e / R0);
        return 1;
    }
    if (where == 2 && stage == k) {             // stage:k, reference layout
        if (k == 0) {                           // c*d0 + k0
            unit = e / d0; idx = (int)(e % d0);
        } else if (kind == KIND_MID) {          // (k0*d2 + c2)*d1 + k1
            unit = e / d1; idx = (int)(e % d1);
        } else if (nst == 2) {                  // k0*d1 + k1
            unit = e / d1; idx = (int)(e % d1);
        } else {                                // (k0*d1 + k1)*d2 + k2
            const long long k0 = e / (d1 * d2), k1 = (e / d2) % d1;
            unit = k1 * d0 + k0; idx = (int)(e % d2);
        }
        return 2;
    }
    if (where == 3 && kind == KIND_LAST) {      // natural output index f
        if (nst == 2) {
            unit = e % d0; idx = (int)(e / d0);
        } else {
            const long long k0 = e % d0, k1 = (e / d0) % d1;
            unit = k1 * d0 + k0; idx = (int)(e / (d0 * d1));
        }
        return 3;
    }
    return 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// The strided rows of a first / middle stage as a 3-D tensor of 32-bit words:
//   first : [c (R0 elems), j (d0), b (batch)]        element (b, j, c) at b n + j R0 + c
//   middle: [c2 (d2 elems), j (d1), (b, k0) (B d0)]  element at (b d0 + k0) R0 + j d2 + c2
// boxes of [U elements x min(L, 256) rows x 1].
template <class T>
int encode_rows_tmap(CUtensorMap* map, const void* base, int kind, long long n, long long batch, long long d0,
                     long long d1, long long d2, int U, long long L) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return merr(TFFT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const long long cw = sizeof(C<T>) / 4;
    const long long es = sizeof(C<T>);
    const long long R0 = n / d0;
    cuuint64_t dims[3], strides[2];
    if (kind == KIND_FIRST) {
        dims[0] = cw * R0; dims[1] = d0; dims[2] = batch;
        strides[0] = R0 * es; strides[1] = n * es;
    } else {
        dims[0] = cw * d2; dims[1] = d1; dims[2] = batch * d0;
        strides[0] = d2 * es; strides[1] = R0 * es;
    }
    cuuint32_t box[3] = {(cuuint32_t)(cw * U), (cuuint32_t)(L < 256 ? L : 256), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return merr(TFFT_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return TFFT_OK;
}

std::mutex occ_mu;
std::map<const void*, int> occ;

int blocks_per_sm(const void* fn, int threads, int smem, int* nb) {
    std::lock_guard<std::mutex> lk(occ_mu);
    auto it = occ.find(fn);
    if (it != occ.end()) {
        *nb = it->second;
        return TFFT_OK;
    }
    if (smem > 48 * 1024) MCU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int v = 0;
    MCU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, threads, smem));
    if (v < 1) return merr(TFFT_EUNSUPPORTED, "pass kernel does not fit on an SM");
    occ[fn] = v;
    *nb = v;
    return TFFT_OK;
}

template <class T>
int launch_pass(const MultiPlan& mp, const PassEntry* pe, int kind, int abft, PassArgs<T>& a, int num_sms,
                cudaStream_t st) {
    const void* fn = pe->fn[kind][abft];
    if (!fn) return merr(TFFT_EUNSUPPORTED, "pass variant not built");
    int nb = 0;
    int rc = blocks_per_sm(fn, pe->threads, pe->smem, &nb);
    if (rc) return rc;
    const long long total = a.batch * a.tiles_per_sig;
    long long grid = std::min<long long>(total, (long long)nb * num_sms);
    if (grid < 1) grid = 1;
    void* args[] = {&a};
    MCU((tfft::note_launch(), cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(pe->threads), args, pe->smem, st)));
    return TFFT_OK;
}

template <class T>
int multi_launch_t(MultiPlan& mp, const MultiLaunch& m, cudaStream_t st) {
    const long long n = mp.n;
    const int nst = mp.nst;
    const long long d0 = mp.d[0], d1 = mp.d[1], d2 = mp.d[2];
    const long long R0 = n / d0;
    const size_t es = sizeof(C<T>);
    const size_t need = m.only_stage >= 0 ? 0 : (size_t)m.batch * n * es;
    if (need > mp.ws_bytes) {
        cudaFree(mp.ws);
        mp.ws = nullptr;
        mp.ws_bytes = 0;
        MCU(cudaMalloc(&mp.ws, need));
        mp.ws_bytes = need;
    }
    const bool abft = m.abft != ABFT_OFF;
    long long tiles[3];
    const PassEntry* pe[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < nst; ++k) {
        pe[k] = pass_entry(mp.prec, lg(mp.d[k]), kind_of(k, nst));
        if (!pe[k]) return merr(TFFT_EUNSUPPORTED, "no pass kernel for stage dim");
        const long long units = k == 0 ? R0 : (k == nst - 1 ? n / mp.d[k] : d0 * d2);
        const int kind = kind_of(k, nst);
        const long long lo_count = kind == KIND_FIRST ? R0 : (kind == KIND_MID ? d2 : d0);
        if (lo_count % pe[k]->u) return merr(TFFT_EUNSUPPORTED, "stage split too narrow for the tile width");
        tiles[k] = units / pe[k]->u;
    }
    T* part_in = nullptr;
    T* part_out = nullptr;
    if (abft) {
        const size_t pb = (size_t)m.batch * (tiles[0] * 3 + tiles[nst - 1] * 2) * sizeof(T);
        if (pb > mp.part_bytes) {
            cudaFree(mp.part);
            mp.part = nullptr;
            mp.part_bytes = 0;
            MCU(cudaMalloc(&mp.part, pb));
            mp.part_bytes = pb;
        }
        part_in = (T*)mp.part;
        part_out = part_in + (size_t)m.batch * tiles[0] * 3;
    }

    if (m.faults && m.nfaults > 0) {  // batched campaign: one fault table per pass
        std::vector<FaultRec> tab((size_t)nst * m.nfaults);
        for (int k = 0; k < nst; ++k) {
            for (long long r = 0; r < m.nfaults; ++r) {
                const HostFault& f = m.faults[r];
                FaultRec& fr = tab[(size_t)k * m.nfaults + r];
                memset(&fr, 0, sizeof(fr));
                if (f.where == 0) continue;
                long long unit = 0;
                int idx = 0;
                fr.where = pass_fault(k, nst, d0, d1, d2, R0, f.where, f.stage, f.elem, unit, idx);
                fr.pos = unit;
                fr.idx = idx;
                fr.signal = (int)f.signal;
                fr.comp = f.comp;
                fr.bit = f.bit;
            }
        }
        const size_t bytes = tab.size() * sizeof(FaultRec);
        if (bytes > mp.ftab_bytes) {
            cudaFree(mp.ftab);
            mp.ftab = nullptr;
            mp.ftab_bytes = 0;
            MCU(cudaMalloc(&mp.ftab, bytes));
            mp.ftab_bytes = bytes;
        }
        MCU(cudaMemcpyAsync(mp.ftab, tab.data(), bytes, cudaMemcpyHostToDevice, st));
        MCU(cudaStreamSynchronize(st));
    }
    for (int k = 0; k < nst; ++k) {
        if (m.only_stage >= 0 && k != m.only_stage) continue;
        const int kind = k == 0 ? KIND_FIRST : (k == nst - 1 ? KIND_LAST : KIND_MID);
        PassArgs<T> a;
        memset(&a, 0, sizeof(a));
        a.batch = m.batch;
        a.sig_base = m.sig_base;
        a.n = n;
        a.in = (const C<T>*)(k == 0 || m.only_stage >= 0 ? m.in : mp.ws);
        a.out = (C<T>*)(k == nst - 1 || m.only_stage >= 0 ? m.out : mp.ws);
        a.tiles_per_sig = tiles[k];
        a.twL = (const C<T>*)mp.twL[k];
        a.inverse = m.inverse;
        a.scale_inv = m.scale_inv;
        a.scale = T(1) / T(n);
        if (kind == KIND_FIRST) {
            a.lo_count = R0; a.in_hi = 0; a.in_lo = 1; a.in_j = R0;
            a.out_hi = 0; a.out_lo = 1; a.out_k = R0;
            a.M = n;
        } else if (kind == KIND_MID) {
            a.lo_count = d2; a.in_hi = R0; a.in_lo = 1; a.in_j = d2;
            a.out_hi = R0; a.out_lo = 1; a.out_k = d2;
            a.M = d1 * d2;
        } else if (nst == 2) {
            a.lo_count = d0; a.in_hi = 0; a.in_lo = R0; a.in_j = 1;
            a.out_hi = 0; a.out_lo = 1; a.out_k = d0;
        } else {
            a.lo_count = d0; a.in_hi = d2; a.in_lo = R0; a.in_j = 1;
            a.out_hi = d0; a.out_lo = 1; a.out_k = d0 * d1;
        }
        if (kind != KIND_LAST) {
            a.ptw_lo = (const C<T>*)mp.ptw_lo[k];
            a.ptw_hi = (const C<T>*)mp.ptw_hi[k];
            a.ptw_shift = mp.ptw_shift[k];
            a.ptw_mask = a.M - 1;
        }
        int abft_v = ABFT_OFF;
        if (abft && kind == KIND_FIRST) {
            // input side: the Wang row in closed form (no table traffic) where it
            // measured faster — L >= 256 and a small batch, whose table reads are
            // a large share of the pass (profiles/etw_cf_r02.txt); otherwise, and
            // for every other encoding, the e^T W row read from the table
            static const long long cf_maxb = [] {
                const char* e = getenv("TFFT_ETW_CF_MAXB");  // A/B override
                return e ? atoll(e) : 8LL;
            }();
            const bool cf = m.abft == ABFT_WANG && d0 >= 256 && m.batch <= cf_maxb;
            abft_v = cf ? ABFT_WANG : ABFT_TABLE;
            a.etw = (const C<T>*)m.etw;
            a.part = part_in;
        } else if (abft && kind == KIND_LAST) {
            abft_v = m.abft;
            a.values = (const C<T>*)m.values;
            a.part = part_out;
        }
        // fault for this pass
        if (m.f_where != 0) {
            a.f_signal = m.f_signal;
            a.f_comp = m.f_comp;
            a.f_bit = m.f_bit;
            long long unit = 0;
            int idx = 0;
            a.f_where = pass_fault(k, nst, d0, d1, d2, R0, m.f_where, m.f_stage, m.f_elem, unit, idx);
            a.f_unit = unit;
            a.f_idx = idx;
        }
        if (m.faults && m.nfaults > 0) {
            a.f_table = (const FaultRec*)mp.ftab + (size_t)k * m.nfaults;
            a.f_div = m.f_div;
        }
        if (pe[k]->pf >= 3 && kind != KIND_LAST) {
            int rc = encode_rows_tmap<T>(&a.tmap, a.in, kind, n, m.batch, d0, d1, d2, pe[k]->u, mp.d[k]);
            if (rc) return rc;
            if (pe[k]->pf == 4 && kind == KIND_FIRST && abft_v != ABFT_OFF) {
                rc = encode_rows_tmap<T>(&a.tmap_etw, m.etw, kind, n, 1, d0, d1, d2, pe[k]->u, mp.d[k]);
                if (rc) return rc;
            }
        }
        int rc = launch_pass<T>(mp, pe[k], kind, abft_v, a, mp.num_sms, st);
        if (rc) return rc;
    }
    if (abft) {
        FinalArgs<T> f;
        memset(&f, 0, sizeof(f));
        f.batch = m.batch;
        f.sig_base = m.sig_base;
        f.part_in = part_in;
        f.tiles_in = tiles[0];
        f.part_out = part_out;
        f.tiles_out = tiles[nst - 1];
        f.delta = (T)m.delta;
        f.abs_floor = (T)m.abs_floor;
        f.floor_coef = sizeof(T) == 4 ? (T)1e-6f : (T)1e-12;
        f.flag_count = m.flag_count;
        f.flag_rec = m.flag_rec;
        f.flag_cap = m.flag_cap;
        f.flag_ovf = m.flag_ovf;
        f.max_key = (typename KeyT<T>::type*)m.max_key;
        f.rel_out = (T*)m.rel_out;
        if (tiles[0] >= 1024) {  // few signals, many tiles: a CTA per signal
            const long long grid = std::min<long long>(m.batch, 4LL * mp.num_sms);
            tfft::note_launch(), abft_finalize_cta_kernel<T><<<(unsigned)std::max<long long>(grid, 1), 256, 0, st>>>(f);
        } else {                 // a warp per signal
            const long long grid = std::min<long long>((m.batch + 7) / 8, 4LL * mp.num_sms);
            tfft::note_launch(), abft_finalize_kernel<T><<<(unsigned)std::max<long long>(grid, 1), 256, 0, st>>>(f);
        }
        MCU(cudaGetLastError());
    }
    return TFFT_OK;
}

}  // namespace

const char* multi_last_error() { return m_err.c_str(); }

int pass_tune_variants(int prec, int logl) {
    int n = 0;
    while (pass_variant(prec, logl, n)) ++n;
    return n;
}

int pass_tune_select(int prec, int logl, int kind, int variant) {
    if ((prec != TFFT_FP32 && prec != TFFT_FP64) || logl < 1 || logl >= 12 || kind < 0 || kind > 2)
        return merr(TFFT_EINVAL, "bad pass selector");
    if (variant >= 0 && !pass_variant(prec, logl, variant)) return merr(TFFT_EINVAL, "no such pass variant");
    g_pass_override[prec][logl][kind] = variant < 0 ? 0 : variant + 1;
    return TFFT_OK;
}

int multi_plan_init(MultiPlan& mp, long long n, int prec, int nst, const int64_t* dims, int num_sms) {
    mp.prec = prec;
    mp.nst = nst;
    mp.n = n;
    mp.num_sms = num_sms;
    if (nst < 2) return merr(TFFT_EUNSUPPORTED, "multi-pass plan needs >= 2 stages");
    for (int k = 0; k < nst; ++k) mp.d[k] = dims[k];
    const long long R0 = n / mp.d[0];
    for (int k = 0; k < nst; ++k) {
        const int kind = kind_of(k, nst);
        const PassEntry* pe = pass_entry(prec, lg(mp.d[k]), kind);
        if (!pe) return merr(TFFT_EUNSUPPORTED, "no pass kernel for stage dim");
        const long long lo_count = kind == KIND_FIRST ? R0 : (kind == KIND_MID ? mp.d[2] : mp.d[0]);
        if (lo_count % pe->u) return merr(TFFT_EUNSUPPORTED, "stage split too narrow for the tile width");
        int rc = upload_multires(prec, mp.d[k], &mp.twL[k]);
        if (rc) return rc;
        if (kind != KIND_LAST) {
            const long long M = kind == KIND_FIRST ? n : mp.d[1] * mp.d[2];
            const int lm = lg(M);
            const int s = (lm + 1) / 2;
            mp.ptw_shift[k] = s;
            rc = upload_roots(prec, M, 1ll << s, 1, &mp.ptw_lo[k]);
            if (rc) return rc;
            rc = upload_roots(prec, M, M >> s, 1ll << s, &mp.ptw_hi[k]);
            if (rc) return rc;
        }
    }
    return TFFT_OK;
}

void multi_plan_free(MultiPlan& mp) {
    for (int k = 0; k < 3; ++k) { cudaFree(mp.twL[k]); mp.twL[k] = nullptr; }
    for (int k = 0; k < 2; ++k) {
        cudaFree(mp.ptw_lo[k]); cudaFree(mp.ptw_hi[k]);
        mp.ptw_lo[k] = mp.ptw_hi[k] = nullptr;
    }
    cudaFree(mp.ws); mp.ws = nullptr; mp.ws_bytes = 0;
    cudaFree(mp.part); mp.part = nullptr; mp.part_bytes = 0;
    cudaFree(mp.ftab); mp.ftab = nullptr; mp.ftab_bytes = 0;
}

int multi_launch_stage(MultiPlan& mp, int k, const void* in, void* out, long long batch, int inverse,
                       cudaStream_t st) {
    if (k < 0 || k >= mp.nst) return merr(TFFT_EINVAL, "stage index out of range");
    MultiLaunch m;
    memset(&m, 0, sizeof(m));
    m.in = in;
    m.out = out;
    m.batch = batch;
    m.inverse = inverse;
    m.abft = ABFT_OFF;
    m.only_stage = k;
    return multi_launch(mp, m, st);
}

int multi_launch(MultiPlan& mp, const MultiLaunch& m, cudaStream_t st) {
    if (m.batch == 0) return TFFT_OK;
    return mp.prec == TFFT_FP32 ? multi_launch_t<float>(mp, m, st) : multi_launch_t<double>(mp, m, st);
}

}  // namespace tfft
