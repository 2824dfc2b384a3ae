// Host-side engine of the B200 hQDWH path: tree, device HODLR storage,
// descriptor arena, workspace and the plan builders for every HODLR operation.
#pragma once

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace spg {

// ---------------------------------------------------------------- tree
// PartitionTree (tree.hpp:12-56): preorder nodes, split at ceil(size/2) while size > n_min.
struct HTree {
    int n = 0, nmin = 0, depth = 0;
    std::vector<int> begin, size, left, right, level, parent, leaf_ord;
    std::vector<int> leaves;                      // preorder ids of leaves, ascending begin
    std::vector<std::vector<int>> internal_at;    // internal nodes per tree depth
    HTree(int n, int nmin);
    int nnodes() const { return (int)begin.size(); }
    bool leaf(int i) const { return left[i] < 0; }
    // all internal nodes / leaves of the subtree rooted at r (preorder)
    void subtree(int r, std::vector<int>& internal, std::vector<int>& lvs) const;
private:
    int build(int b, int s, int lev, int par);
};

// ---------------------------------------------------------------- device arena
// Descriptor arrays are staged on the host and uploaded once; device addresses
// are fixed at plan time so a plan can be replayed (or graph-captured).
class Arena {
public:
    explicit Arena(size_t bytes);
    ~Arena();
    template <class T>
    T* push(const std::vector<T>& v) {
        if (v.empty()) return nullptr;
        return static_cast<T*>(push_raw(v.data(), sizeof(T) * v.size()));
    }
    void* push_raw(const void* src, size_t bytes);
    void commit(cudaStream_t st);   // upload everything staged since the last commit
    size_t used() const { return off_; }
    void reset() { off_ = 0; committed_ = 0; }
    // descriptors pushed after a mark can be dropped again once their launches are done
    // (the descriptors of captured graphs stay below the mark)
    size_t mark() const { return off_; }
    void release(size_t m) { off_ = m; committed_ = std::min(committed_, m); }
private:
    char* dev_ = nullptr;
    size_t cap_ = 0, off_ = 0, committed_ = 0;
    std::vector<char> host_;
};

// stack allocator over one big device buffer (doubles); stream order makes reuse safe
class Workspace {
public:
    explicit Workspace(size_t ndoubles);
    ~Workspace();
    double* base() const { return base_; }
    long long alloc(long long n);   // returns offset (doubles)
    double* ptr(long long off) const { return base_ + off; }
    long long mark() const { return top_; }
    void release(long long m) { top_ = m; }
    long long peak() const { return peak_; }
    size_t capacity() const { return cap_; }
private:
    double* base_ = nullptr;
    size_t cap_ = 0;
    long long top_ = 0, peak_ = 0;
};

// ---------------------------------------------------------------- device HODLR
// Level-ordered packed storage: leaves packed column-major;
// per tree depth t one U slab and one V slab of n x KCAP (column-major, ld n).
// Node x at depth t: upper.U = U_t[rows of left(x)], upper.V = V_t[rows of right(x)],
//                    lower.U = U_t[rows of right(x)], lower.V = V_t[rows of left(x)].
struct DHodlr {
    DHodlr() = default;
    DHodlr(const DHodlr&) = delete;
    DHodlr& operator=(const DHodlr&) = delete;
    ~DHodlr() { release(); }
    const HTree* t = nullptr;
    double* leaves = nullptr;
    long long* d_leaf_off = nullptr;
    std::vector<long long> leaf_off;
    double* U = nullptr;
    double* V = nullptr;
    int* rank = nullptr;
    double* dinv = nullptr;                 // diagonal-block inverses (used when this is a triangular factor)
    // triangular factors only: per node y the solved coupling bases (see Engine::op_solve_prep)
    //   tV_t[rows r(y)] = W_{r(y)}^{-T} V_y   and   tU_t[rows l(y)] = W_{l(y)}^{-1} U_y
    double* tU = nullptr;
    double* tV = nullptr;
    bool tready = false;                    // plan-build-time flag: tU / tV are current
    std::vector<char> tv_built;             // plan-build-time: tV of these nodes built by the Cholesky
    double* tslabU(int lev) const { return tU + (size_t)lev * KCAP * t->n; }
    double* tslabV(int lev) const { return tV + (size_t)lev * KCAP * t->n; }
    long long* d_dinv_off = nullptr;
    std::vector<long long> dinv_off;
    size_t leaf_doubles = 0, slab_doubles = 0;
    void alloc(const HTree& tree, Arena& arena);
    void release();
    double* leaf(int id) const { return leaves + leaf_off[t->leaf_ord[id]]; }
    double* slabU(int lev) const { return U + (size_t)lev * KCAP * t->n; }
    double* slabV(int lev) const { return V + (size_t)lev * KCAP * t->n; }
    double* upU(int id) const { return slabU(t->level[id]) + t->begin[t->left[id]]; }
    double* upV(int id) const { return slabV(t->level[id]) + t->begin[t->right[id]]; }
    double* loU(int id) const { return slabU(t->level[id]) + t->begin[t->right[id]]; }
    double* loV(int id) const { return slabV(t->level[id]) + t->begin[t->left[id]]; }
    int* rup(int id) const { return rank + 2 * id; }
    int* rlo(int id) const { return rank + 2 * id + 1; }
    double* leaf_dinv(int id) const { return dinv + dinv_off[t->leaf_ord[id]]; }
    DevHodlrView view() const { return {leaves, d_leaf_off, U, V, rank, t->n, dinv, d_dinv_off}; }
    void zero(cudaStream_t st) const;
};

// a global-row-indexed panel: rows [0, n), KCAP columns, ld n
struct Panel {
    double* p = nullptr;
    int ld = 0;
    double* at(int row) const { return p + row; }
};

using Launch = std::function<void(cudaStream_t)>;

struct Plan {
    std::vector<Launch> launches;
    void run(cudaStream_t st) const { for (auto& l : launches) l(st); }
    size_t size() const { return launches.size(); }
};

// ---------------------------------------------------------------- the engine
struct Scalars {          // device scalar block
    double* scal;         // [0] alpha [1] l0 [2] 1/alpha
    double* slots;        // per-iteration coefficients (see launch_iter_params)
    double* sched;        // 4 * 64
    int* count;
    int* counter;
    unsigned* status;     // status word + overflow diagnostics (16 ints)
    double* counters;     // [0] recompression bytes 8(p+s)(k_in+k_out) [1] GEMM flops 2MNK [2] truncation tasks
                          // [3] core statistics [4] truncation QR flops [5] core + basis flops (8 doubles)
};

// kernel classes timed with CUDA events in profile mode
enum ProfClass { PC_TRUNC = 0, PC_GEMM, PC_HSOLVE, PC_LEAF, PC_NCLS };

void launch_zero_lower_ranks(int* rank, int nnodes, cudaStream_t st);
void launch_phase_mark(const double* counters, double* snap, double* acc, int phase, int end, cudaStream_t st);

class Engine {
public:
    Engine(int n, int nmin, double eps, size_t ws_doubles = 0);
    ~Engine();
    const HTree& tree() const { return tree_; }
    Arena& arena() { return *arena_; }
    Workspace& ws() { return *ws_; }
    cudaStream_t stream() const { return st_; }
    Scalars& sc() { return sc_; }
    double eps() const { return eps_; }
    DevTree dtree() const { return dtree_; }

    // ---- plan builders (append launches to `p`) ------------------------------
    // truncation batch (lowrank.hpp:67-86); tasks' workspace is assigned here
    void trunc(Plan& p, std::vector<TTask> tasks);
    void trunc_batch(Plan& p, std::vector<TTask> tasks, Workspace& wsp, bool release);
    void gemm(Plan& p, std::vector<GemmItem> items, const std::vector<int3>& caps);
    // Y = H|_sub X (trans: H|_sub^T X) for each request (apply_rec/applyT_rec, hodlr.hpp:202-249)
    struct ApplyReq { const DHodlr* H; int root; int trans; const double* X; const int* ncp; double* Y; };
    void apply(Plan& p, const std::vector<ApplyReq>& reqs);
    // add_lowrank_into (hodlr.hpp:400-405) of s * QU QV^T into the subtrees (batched, disjoint)
    struct Cascade { int root; const double* QU; const double* QV; const int* qrank; double s; };
    void cascade(Plan& p, DHodlr& H, const std::vector<Cascade>& cs, bool upper_only = false);
    void hsolve(Plan& p, const DHodlr& W, std::vector<HSolveItem> items);
    // the same solves, subtree-parallel: all leaves at once, then one batched low-rank
    // correction per tree level with the solved coupling bases (needs op_solve_prep(W))
    void psolve(Plan& p, const DHodlr& W, const std::vector<HSolveItem>& items);
    void copy(Plan& p, std::vector<CopyItem> items, int maxm, int maxk);
    void leaf_trsm_batch(Plan& p, const std::vector<TrsmItem>& ti, const std::vector<int2>& ct);

    // ---- HODLR operations (hodlr.hpp) ------------------------------------------
    void op_axpby(Plan& p, double a, const double* ap, const DHodlr& A, double b, const double* bp, const DHodlr& B,
                  DHodlr& C);
    void op_symmetrize(Plan& p, DHodlr& H);
    void op_scale_shift(Plan& p, DHodlr& H, double s, const double* sp, double mu);
    void op_copy(Plan& p, const DHodlr& src, DHodlr& dst);
    // inverses of the 32x32 diagonal blocks of every leaf of an upper-triangular factor
    void op_leaf_dinv(Plan& p, DHodlr& W);
    // solved coupling bases tU / tV of a finished upper-triangular factor (bottom-up)
    void op_solve_prep(Plan& p, DHodlr& W);
    void op_multiply(Plan& p, const DHodlr& A, const DHodlr& B, DHodlr& C, bool upper_only = false);
    // defer_trunc: W12 = trunc(W11^{-T} M12) is taken off the critical path (own stream)
    // and the Schur complement uses the untruncated pair (differs at the eps level)
    void op_cholesky(Plan& p, const DHodlr& M, DHodlr& W, DHodlr& work, bool defer_trunc = false);
    void op_solve_upper_right(Plan& p, const DHodlr& B, const DHodlr& W, DHodlr& Y, DHodlr& work);
    void op_solve_upperT_right(Plan& p, const DHodlr& B, const DHodlr& W, DHodlr& Y, DHodlr& work);

    std::unique_ptr<DHodlr> new_hodlr();

    // profile mode: every batch is bracketed by a pair of CUDA events (plans are then not replayed)
    void set_profile(bool on) { profile_ = on; }
    bool profile() const { return profile_; }
    void prof_sum(double* ms_per_class, long long* batches_per_class) const;
    void prof_clear();
    void push_timed(Plan& p, int cls, Launch l);
    void push(Plan& p, Launch l);
    void record(Plan& p, int e);   // event slot e
    void wait(Plan& p, int e);
    // Race diagnostics (SPG_DBG_HASHLOG=1): an order-independent checksum of a just-written region,
    // computed by a small kernel queued on the stream of the current mode, into the next log slot.
    // The log of a run (dump_hashlog) names, in plan order, every intermediate result of the
    // H-Cholesky; the first slot that differs between two runs is where they part.
    void hash_region(Plan& p, const char* tag, int node, const double* ptr, int rows, int cols, int ld,
                     const int* rankp);
    void dump_hashlog(cudaStream_t st);

private:
    unsigned long long* hashlog_ = nullptr;
    std::vector<std::string> hashtags_;
    void chol_rec(Plan& p, int x, DHodlr& M, DHodlr& W);
    void sur_rec(Plan& p, int x, DHodlr& B, const DHodlr& W, DHodlr& Y);
    void surt_rec(Plan& p, int x, DHodlr& B, const DHodlr& W, DHodlr& Y);
    void sur_levels(Plan& p, DHodlr& B, const DHodlr& W, DHodlr& Y);
    void surt_levels(Plan& p, DHodlr& B, const DHodlr& W, DHodlr& Y);
    double* panel(int which);   // persistent global-row panels (n x KCAP)

    HTree tree_;
    double eps_;
    cudaStream_t st_ = nullptr;
    std::vector<cudaStream_t> sides_;   // deferred Schur cascades of the Cholesky (per depth + leaves)
    int side_sel_ = -1;                 // stream of the launches being built (-1 = main)
    std::vector<cudaEvent_t> events_;
    std::vector<std::unique_ptr<Workspace>> ws_side_;   // one stack per side stream
    std::vector<double*> chol_panels_;  // per-depth Schur panels (a deferred cascade reads its own)
    bool chol_deferred_ = false;
    bool chol_defer_trunc_ = false;
    int ncasc_ = 0;                     // cascade side streams (depth streams + the leaf stream)
    int wtr_idx_ = 0;                   // side stream of the deferred W12 truncations
    int ev_base2_ = 0;                  // event slots: x-ready(x) = ev_base2_ + x, w12-done(x) = ev_base2_ + nn + x
    int wtr_last_ev_ = -1;              // latest W12 truncation event (FIFO stream: covers all earlier ones)
    int tv_idx_ = 0;                    // side stream building the Cholesky's tV bases
    int ev_base3_ = 0;                  // chol(x) done = ev_base3_ + x, tV_x built = ev_base3_ + nn + x
    bool chol_tv_ = false;
    std::vector<char> tv_need_;
    std::vector<double*> xpanels_;      // per-depth untruncated W11^{-T} M12.U panels
    double* leaf_scr_ = nullptr;        // Schur block of a split leaf Cholesky (main stream only)
    std::vector<int> last_leaf_ev_, last_block_ev_;   // latest side-stream event touching a leaf / block
    void cascade_chol(Plan& p, DHodlr& M, int x, int root, const double* QU, const double* QV, const int* qrank);
    void leaf_chol_split(Plan& p, const double* Ml, double* Wl, double* D, int s);
    std::unique_ptr<Arena> arena_;
    std::unique_ptr<Workspace> ws_;
    DevTree dtree_{};
    Scalars sc_{};
    double* scalar_mem_ = nullptr;
    double* host_pinned_ = nullptr;   // page-locked 64 doubles for asynchronous scalar read-back
public:
    double* host_pinned() const { return host_pinned_; }
private:
    std::vector<double*> panels_;
    double* coef_ = nullptr;    // per-node coefficient blocks (KCAP x KCAP)
    double* pcoef_ = nullptr;   // per-node psolve coupling products (KCAP x KCAP)
    int* iranks_ = nullptr;     // scratch ranks (4 * nnodes)
    std::vector<std::unique_ptr<DHodlr>> owned_;
    int cur_op_ = 0;
    bool profile_ = false;
    struct ProfRec { int cls, op; cudaEvent_t a, b; int ntask, rows, side; };
    int prof_ntask_ = 0, prof_rows_ = 0;   // shape of the next timed truncation batch
    std::vector<ProfRec> prof_;
};

}  // namespace spg
