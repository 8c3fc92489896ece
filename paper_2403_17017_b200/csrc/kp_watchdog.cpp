// kp_watchdog.cpp -- failure detection for the row-sharded path ("ncclCommGetAsyncError
// polling with a timeout").  A native thread polls the communicator's asynchronous error state
// and a host heartbeat; on an NCCL error, or when no heartbeat arrived within the timeout (a
// hung collective / peer), it aborts the communicator (ncclCommAbort), which makes the blocked
// collective kernels return so the rank can fail loudly instead of hanging the node.
//
// NCCL is not linked: the symbols are resolved from the libnccl.so.2 the process already
// loaded (torch's), so the library carries no NCCL build dependency.
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <thread>

#include "../../include/kernelpick_b200.h"

namespace {

typedef int (*GetAsyncErrorFn)(void *, int *);
typedef int (*AbortFn)(void *);
typedef const char *(*ErrorStringFn)(int);

constexpr int kNcclSuccess = 0;
constexpr int kNcclInProgress = 7;

int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace

struct kp_watchdog {
    void *comm = nullptr;
    GetAsyncErrorFn get_error = nullptr;
    AbortFn abort_comm = nullptr;
    ErrorStringFn error_string = nullptr;
    int64_t timeout_ns = 0, poll_ns = 0;
    std::atomic<int64_t> last_beat{0};
    std::atomic<int> state{KP_WD_OK};
    std::atomic<int> nccl_result{0};
    std::atomic<bool> stop{false};
    std::thread th;

    void run() {
        while (!stop.load(std::memory_order_acquire)) {
            std::this_thread::sleep_for(std::chrono::nanoseconds(poll_ns));
            int r = kNcclSuccess;
            const int rc = get_error(comm, &r);
            if (rc != kNcclSuccess || (r != kNcclSuccess && r != kNcclInProgress)) {
                nccl_result.store(rc != kNcclSuccess ? rc : r);
                state.store(KP_WD_NCCL_ERROR);
                abort_comm(comm);
                return;
            }
            if (timeout_ns > 0 && now_ns() - last_beat.load(std::memory_order_acquire) > timeout_ns) {
                state.store(KP_WD_TIMEOUT);
                abort_comm(comm);
                return;
            }
        }
    }
};

extern "C" {

KP_API int kp_watchdog_start(void *nccl_comm, int64_t timeout_ms, int64_t poll_ms, kp_watchdog **out) {
    if (!nccl_comm || !out || timeout_ms < 0 || poll_ms <= 0) return KP_EINVAL;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return KP_EUNSUPPORTED;
    kp_watchdog *w = new kp_watchdog();
    w->get_error = (GetAsyncErrorFn)dlsym(h, "ncclCommGetAsyncError");
    w->abort_comm = (AbortFn)dlsym(h, "ncclCommAbort");
    w->error_string = (ErrorStringFn)dlsym(h, "ncclGetErrorString");
    if (!w->get_error || !w->abort_comm) {
        delete w;
        return KP_EUNSUPPORTED;
    }
    w->comm = nccl_comm;
    w->timeout_ns = timeout_ms * 1000000;
    w->poll_ns = poll_ms * 1000000;
    w->last_beat.store(now_ns());
    w->th = std::thread([w] { w->run(); });
    *out = w;
    return KP_OK;
}

KP_API int kp_watchdog_heartbeat(kp_watchdog *w) {
    if (!w) return KP_EINVAL;
    w->last_beat.store(now_ns(), std::memory_order_release);
    return w->state.load();
}

KP_API int kp_watchdog_status(kp_watchdog *w, int32_t *nccl_result, char *msg, size_t msg_len) {
    if (!w) return KP_EINVAL;
    const int s = w->state.load();
    if (nccl_result) *nccl_result = w->nccl_result.load();
    if (msg && msg_len) {
        const char *t = s == KP_WD_OK ? "ok"
                        : s == KP_WD_TIMEOUT ? "no heartbeat within the timeout: communicator aborted"
                        : (w->error_string ? w->error_string(w->nccl_result.load()) : "NCCL asynchronous error");
        strncpy(msg, t, msg_len - 1);
        msg[msg_len - 1] = 0;
    }
    return s;
}

KP_API int kp_watchdog_stop(kp_watchdog *w) {
    if (!w) return KP_EINVAL;
    w->stop.store(true, std::memory_order_release);
    if (w->th.joinable()) w->th.join();
    const int s = w->state.load();
    delete w;
    return s;
}

}  // extern "C"
