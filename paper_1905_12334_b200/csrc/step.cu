// step.cu -- fp8b_dense_step: one quantized Dense-layer training step on device.
//
// The caller of the hot path in the reference is nn::Network (nn.cpp:155-458)
// driven by train() (nn.cpp:540-547). For a Dense layer that is six Q nodes,
// three gemm_fp8 calls, a finiteness check, two update_tensor calls and a
// LossScaler::step, with a full FP32 tensor materialised between each. Here the
// output Q nodes are fused into the GEMM epilogues, the finiteness check is the
// Q kernels' own counters, the update skips itself on device and also emits the
// next step's E5M2 weights, the gate merge and the scaler step ride on the last
// update kernel, and the scaler state never leaves HBM: 7 kernel launches (9 with
// a bias; no memset nodes -- each costs ~4 us on a captured graph's critical
// path), no host synchronisation, CUDA-graph capturable.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace fp8b {
// counters[0..5] = 0, fwd[0..2] = 0 (fwd may be null)
__global__ void zero_counters_kernel(int64_t* counters, int64_t* fwd) {
    pdl_trigger();
    if (threadIdx.x < 6) counters[threadIdx.x] = 0;
    else if (threadIdx.x < 9 && fwd) fwd[threadIdx.x - 6] = 0;
}

// Side streams for the step's independent branches. Given Q(X) and Q(E), the
// three GEMMs of the layer are independent (fprop reads qx and w_q, bprop qe and
// w_q, wgrad qx and qe) and together need 64 of the 148 SMs at config-1 size, so
// they run side by side: main = Q(X) -> fprop, side 0 = Q(E) -> bprop, side 1 =
// wgrad once both Q nodes are done. Fork / join go through events, which
// CUDA-graph capture turns into parallel graph branches. One set per host
// thread and device, so concurrent callers on different streams never share
// events.
struct SideStream {
    cudaStream_t s[2] = {nullptr, nullptr};
    cudaEvent_t fork = nullptr, qx = nullptr, qe = nullptr, join[2] = {nullptr, nullptr};
    int dev = -1;
};
// nullptr -> run every branch on the caller's stream (no fork). That is also
// the path when the first call of a thread is inside a stream capture, where
// creating the streams / events is not allowed.
static SideStream* side_stream(cudaStream_t caller) {
    thread_local SideStream ss[16];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
    SideStream& x = ss[dev];
    if (x.dev != dev) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(caller, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
            return nullptr;
        bool ok = true;
        for (int i = 0; i < 2; ++i)
            ok = ok && cudaStreamCreateWithFlags(&x.s[i], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&x.join[i], cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&x.qx, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&x.qe, cudaEventDisableTiming) == cudaSuccess;
        if (!ok) return nullptr;
        x.dev = dev;
    }
    return &x;
}
}  // namespace fp8b

extern "C" {

int fp8b_dense_step(const fp8b_dense_step_t* s, void* stream) {
    if (!s) return FP8B_EINVAL;
    const int64_t B = s->batch, I = s->in_features, O = s->out_features;
    if (B <= 0 || I <= 0 || O <= 0 || !s->x || !s->e || !s->w_master || !s->w_momentum ||
        !s->w_q || !s->qx || !s->qy || !s->qe || !s->qdw || !s->counters || !s->gate ||
        !s->scaler)
        return FP8B_EINVAL;
    if (s->b_master && (!s->b_momentum || !s->b_value || !s->db)) return FP8B_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int rc;
#define FP8B_TRY(expr)          \
    do {                        \
        rc = (expr);            \
        if (rc) return rc;      \
    } while (0)
    // one tiny kernel instead of two memset nodes: in a captured graph every
    // node on the critical path costs ~3 us of dependent-launch latency (the
    // step measured 29 us with the two memsets, 20 us with none)
    fp8b::zero_counters_kernel<<<1, 32, 0, st>>>(s->counters, s->fwd_counters);
    if (cudaGetLastError() != cudaSuccess) return FP8B_ECUDA;
    fp8b::note_launches(1);
    fp8b_quant_config_t rne{};
    rne.mode = FP8B_RNE;
    rne.seed = 1;
    rne.saturate = s->saturate;
    fp8b::SideStream* ss = fp8b::side_stream(st);
    void* side0 = ss ? (void*)ss->s[0] : stream;
    void* side1 = ss ? (void*)ss->s[1] : stream;
    // Open forks are always joined, also on the early-return paths (FP8B_TRY):
    // under stream capture an unjoined fork would invalidate the capture, and run
    // eagerly the side-stream work would stay unordered with the caller's later
    // work.
    struct Branch {
        fp8b::SideStream* ss;
        cudaStream_t st;
        bool open = false;
        bool fork() {
            if (!ss) return true;
            if (cudaEventRecord(ss->fork, st) != cudaSuccess ||
                cudaStreamWaitEvent(ss->s[0], ss->fork, 0) != cudaSuccess ||
                cudaStreamWaitEvent(ss->s[1], ss->fork, 0) != cudaSuccess)
                return false;
            open = true;
            return true;
        }
        bool join() {
            if (!ss || !open) return true;
            open = false;
            bool ok = true;
            for (int i = 0; i < 2; ++i)
                ok = (cudaEventRecord(ss->join[i], ss->s[i]) == cudaSuccess &&
                      cudaStreamWaitEvent(st, ss->join[i], 0) == cudaSuccess) && ok;
            return ok;
        }
        ~Branch() { join(); }
    } br{ss, st};
    // ---- side 0: Q(E) (+ db), then bprop (nn.cpp:294-326)
    if (!br.fork()) return FP8B_ECUDA;
    FP8B_TRY(fp8b_quantize(s->e, s->qe, B * O, FP8B_E5M2, &rne, s->counters, side0));
    if (s->b_master) {
        FP8B_TRY(fp8b_bias_grad(s->qe, FP8B_E5M2, B, O, s->db, side0));
        FP8B_TRY(fp8b_count_nonfinite(s->db, O, s->counters, side0));
    }
    if (ss && cudaEventRecord(ss->qe, ss->s[0]) != cudaSuccess) return FP8B_ECUDA;
    fp8b_gemm_args_t g{};
    g.engine = s->engine;
    g.cq_fmt = FP8B_E5M2;
    g.cq_mode = FP8B_RNE;
    g.cq_seed = 1;
    g.cq_saturate = s->saturate;
    if (s->qdx) {
        // bprop: dX[B,I] = qe . w_q^T  (w_q [I,O] read as the K-major [N=I, K=O] operand)
        fp8b_gemm_args_t gb = g;
        gb.a_major = FP8B_K_MAJOR;
        gb.b_major = FP8B_K_MAJOR;
        gb.cq = s->qdx;
        gb.cq_counters = s->counters;
        FP8B_TRY(fp8b_gemm(s->qe, s->w_q, B, I, O, FP8B_E5M2, &gb, side0));
    }
    // ---- main: forward (nn.cpp:187-203): qx = Q(x); y = qx . w_q (+ b); qy = Q(y)
    if (s->b_master) FP8B_TRY(fp8b_dequantize(s->b_master, s->b_value, O, FP8B_FP16, stream));
    FP8B_TRY(fp8b_quantize(s->x, s->qx, B * I, FP8B_E5M2, &rne, s->fwd_counters, stream));
    if (ss && cudaEventRecord(ss->qx, st) != cudaSuccess) return FP8B_ECUDA;
    {
        fp8b_gemm_args_t gf = g;
        gf.a_major = FP8B_K_MAJOR;
        gf.b_major = FP8B_MN_MAJOR;
        gf.c = s->y;
        gf.bias = s->b_master ? s->b_value : nullptr;
        gf.cq = s->qy;
        gf.cq_counters = s->fwd_counters;
        FP8B_TRY(fp8b_gemm(s->qx, s->w_q, B, O, I, FP8B_E5M2, &gf, stream));
    }
    // ---- side 1: wgrad dW[I,O] = qx^T . qe (qx read M-major, qe N-major; no
    // transpose pass), once both Q nodes are done
    if (ss && (cudaStreamWaitEvent(ss->s[1], ss->qx, 0) != cudaSuccess ||
               cudaStreamWaitEvent(ss->s[1], ss->qe, 0) != cudaSuccess))
        return FP8B_ECUDA;
    {
        fp8b_gemm_args_t gw = g;
        gw.a_major = FP8B_MN_MAJOR;
        gw.b_major = FP8B_MN_MAJOR;
        gw.cq = s->qdw;
        gw.cq_counters = s->counters + 3;
        FP8B_TRY(fp8b_gemm(s->qx, s->qe, I, O, B, FP8B_E5M2, &gw, side1));
    }
    if (!br.join()) return FP8B_ECUDA;
    // grads_finite gate (nn.cpp:401-411): overflow of qe/qdw/qdx, NaN in qdw,
    // non-finite db = the sum of the step's two counter sets. The update kernels
    // read both; the last one stores the merged gate (no merge launch).
    // ---- apply_update (nn.cpp:436-458), skipped on device when the gate is set
    fp8b_sgd_args_t u{};
    u.lr = s->lr;
    u.mu = s->mu;
    u.two_lambda = s->two_lambda;
    u.scale = 1.0f;
    u.scaler = s->scaler;
    u.skip_counters = s->counters;
    u.skip_counters2 = s->counters + 3;
    u.master_mode = s->master_mode;
    u.bits = s->bits;
    u.seed = s->seed ? s->seed : 1;
    u.w_e5m2 = s->w_q;
    u.w_saturate = s->saturate;
    // LossScaler::step(grads_finite, iteration) (nn.cpp:547) rides on the step's
    // last update kernel (its last CTA, after every CTA has read the scale)
    u.step_iteration = s->iteration;
    u.step_scaler = s->b_master ? 0 : 1;
    u.gate_out = s->b_master ? nullptr : s->gate;
    FP8B_TRY(fp8b_sgd_momentum_update(s->qdw, FP8B_E5M2, s->w_master, s->w_momentum, I * O, &u,
                                      stream));
    if (s->b_master) {
        u.two_lambda = 0.0f;  // biases are not regularised (nn.cpp:445, 452)
        u.seed = s->seed + 1 ? s->seed + 1 : 1;
        u.w_e5m2 = nullptr;
        u.step_scaler = 1;
        u.gate_out = s->gate;
        FP8B_TRY(fp8b_sgd_momentum_update(s->db, FP8B_F32, s->b_master, s->b_momentum, O, &u,
                                          stream));
    }
#undef FP8B_TRY
    return FP8B_OK;
}

}  // extern "C"
