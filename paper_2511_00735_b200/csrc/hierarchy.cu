// K2 merges: level-by-level Schur elimination of the quadtree merge order.
//
// The reference eliminates level l of the block-sparse system M_l
// (eliminate_level, proj/src/dissection.cpp:153-198) with per-group LUs and
// std::map block updates, M_{l+1} = D - C A^{-1} B.  The level systems are
// exactly box ItI maps scattered into the skeleton:
//     M_l = I + sum_{boxes b of level l} P_b T_b Q_b^T,
// so the B200 path keeps one dense ItI map per box and performs each group
// elimination as a two-box merge (the generalisation of merge_pair,
// dissection.cpp:23-82, to boxes).  For a merge of box 1 (holding the faces'
// e1) and box 2 across separator s, with u_k the incoming data on box k's
// remaining perimeter p_k:
//     x1 = W [T2_ss T1_sp u1 - T2_sp u2],  W = (I - T2_ss T1_ss)^{-1}
//     x2 = -T1_ss x1 - T1_sp u1
//     T_new = [[T1_pp, 0], [0, T2_pp]] + [[T1_ps X1], [T2_ps X2]]
// which is D + C A^{-1} B of the reference restricted to the structurally
// non-zero blocks.  Every merge of a level runs in the same few grouped
// launches: one gather (children permuted to [p | s] order), one copy batch,
// four grouped DMMA GEMMs and one batched inverse.
#include <algorithm>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <unordered_map>

#include "device.cuh"
#include "hierarchy.hpp"
#include "zgemm.hpp"

namespace hpsb {

Hierarchy::~Hierarchy() = default;

namespace {
struct HostBox {
  std::vector<BoxPos> pos;
  const double2* T = nullptr;
  int ld = 0;
};

// HPSB_TRACE=1: host wall time per build phase (stderr), to separate host
// bookkeeping from device time.
struct Trace {
  bool on = std::getenv("HPSB_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  std::vector<std::pair<std::string, double>> acc;
  void mark(const char* name) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - t).count();
    t = now;
    for (auto& kv : acc)
      if (kv.first == name) {
        kv.second += ms;
        return;
      }
    acc.emplace_back(name, ms);
  }
  ~Trace() {
    if (!on) return;
    std::fprintf(stderr, "[hpsb trace hierarchy]");
    for (auto& kv : acc) std::fprintf(stderr, " %s=%.1fms", kv.first.c_str(), kv.second);
    std::fprintf(stderr, "\n");
  }
};

// Host threads for the per-group bookkeeping of a level (independent groups;
// results land in per-group slots, so the outcome does not depend on T).
int host_threads() {
  static const int t = [] {
    const char* e = std::getenv("HPSB_HOST_THREADS");
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, e ? std::atoi(e) : std::min(16, hw > 0 ? hw : 1));
  }();
  return t;
}
template <class F>
void parallel_chunks(int count, int threads, F&& fn) {  // fn(begin, end, thread)
  threads = std::max(1, std::min(threads, count / 256 + 1));
  if (threads == 1) {
    fn(0, count, 0);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        fn(static_cast<int>(static_cast<int64_t>(count) * t / threads),
           static_cast<int>(static_cast<int64_t>(count) * (t + 1) / threads), t);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// Per-group result of the bookkeeping pass.
struct GroupPlan {
  bool own = false;
  int p[2] = {0, 0};
  std::vector<int> perm[2];           // [perimeter | separator] positions (own groups)
  std::vector<BoxPos> cpos[2];        // the child's positions in that order
  std::vector<BoxPos> next_pos;       // merged box perimeter
};
}  // namespace

// pivot = false: the merge inverses use diagonal pivots (InverseBatch
// diag_pivots); *guard_tripped reports a blocked inverse whose diagonal block
// failed the guard, and build_hierarchy then redoes the build with pivoting.
std::unique_ptr<Hierarchy> build_hierarchy_pass(Skeleton* sk, int depth,
                                                const std::function<void(Hierarchy*)>& before_wait,
                                                bool pivot, bool* guard_tripped) {
  Context* ctx = sk->ctx;
  const FaceGraph& g = sk->graph;
  const int total = g.num_levels();
  if (depth == 0) depth = total;
  if (depth < 1 || depth > total) throw InvalidArgument("build_hierarchy: depth out of range");
  auto h = std::make_unique<Hierarchy>();
  h->ctx = ctx, h->sk = sk, h->depth = depth, h->total_levels = total;
  const Elements* el = sk->el;
  const int ne = el->n * el->n, nb = el->nb, m = sk->m, bs = sk->bs;
  // Sharded: levels 1..last_local run on this rank's subtree only; the
  // subtree boxes are then broadcast and the top levels run on every rank.
  const Partition& part = el->part;
  const bool sharded = ctx->world() > 1;
  if (sharded && depth <= part.last_local)
    throw InvalidArgument("build_hierarchy: a sharded hierarchy must reach the global levels (depth > " +
                          std::to_string(part.last_local) + ")");

  // Level-1 boxes are the elements (all 4(N-1) positions, physical ones -1).
  std::vector<HostBox> boxes(ne);
  std::vector<int> elem_box(ne);
  for (int e = 0; e < ne; ++e) {
    boxes[e].pos.resize(nb);
    for (int b = 0; b < nb; ++b)
      boxes[e].pos[b] = {sk->h_in[static_cast<size_t>(e) * nb + b],
                         sk->h_out[static_cast<size_t>(e) * nb + b]};
    boxes[e].T = el->T.p + static_cast<size_t>(e) * nb * nb;
    boxes[e].ld = nb;
    elem_box[e] = e;
  }
  // skeleton index -> position in its box (-1 elsewhere).  The boxes merging
  // at a level own disjoint slots, so the threads of the parallel pass below
  // write disjoint entries of one shared table.
  std::vector<int> pos_of(sk->dim, -1);
  std::vector<int> prev_merge_of;  // previous level: group (= box of this level) -> merge index
  // Rank holding each current box's map (sharded; level 1: the element's
  // owner).  Owner-computes at the global levels: a merge runs on the rank
  // that holds its first child (the box with the faces' e1) and receives the
  // second child from its holder; the coarse level is replicated.
  std::vector<int> box_owner(ne, 0);
  for (int e = 0; e < ne; ++e) box_owner[e] = sharded ? part.elem_owner[e] : 0;
  const std::vector<std::vector<int>> owners = merge_owners(g, part);
  const int me = ctx->rank();
  DevBuf<double2> tnew_prev;  // previous level's merged maps (children of this level)
  DevBuf<int> d_status(2);  // [0] singular pivot tag + 1, [1] diagonal-pivot guard
  HPSB_CUDA(cudaMemsetAsync(d_status.p, 0, 2 * sizeof(int), ctx->stream));

  HPSB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  Trace tr;
  for (int level = 1; level <= depth; ++level) {
    tr.mark("other");
    auto L = std::make_unique<LevelOps>();
    L->level = level;
    L->first_face = g.level_range[level - 1].first;
    L->nfaces = g.num_faces() - L->first_face;
    L->coarse = (level == depth);
    const auto& groups = g.groups[level - 1];
    const int ng = static_cast<int>(groups.size());

    // ---- children in [perimeter | separator] order (parallel over groups)
    std::vector<std::vector<int>> perms;  // per child, positions into its HostBox
    std::vector<const HostBox*> srcs;
    size_t toff = 0;
    std::vector<std::vector<BoxPos>> next_pos(ng);  // merged box perimeter, every group
    std::vector<int> merge_of(ng, -1);              // group -> this rank's merge index
    std::vector<GroupPlan> plan(ng);
    parallel_chunks(ng, host_threads(), [&](int g0, int g1, int) {
      std::vector<char> is_sep[2];
      std::vector<int> sep[2];
      for (int gi = g0; gi < g1; ++gi) {
        GroupPlan& gp = plan[gi];
        const Face& f0 = g.faces[groups[gi][0]];
        gp.own = !sharded || level == depth || box_owner[elem_box[f0.e1]] == me;
        const HostBox* bx[2] = {&boxes[elem_box[f0.e1]], &boxes[elem_box[f0.e2]]};
        for (int k = 0; k < 2; ++k)
          for (int i = 0; i < static_cast<int>(bx[k]->pos.size()); ++i)
            if (bx[k]->pos[i].in >= 0) pos_of[bx[k]->pos[i].in] = i;
        for (int k = 0; k < 2; ++k) {
          is_sep[k].assign(bx[k]->pos.size(), 0);
          sep[k].clear();
        }
        for (int f : groups[gi]) {
          if (g.faces[f].e1 == -1) throw std::logic_error("bad face");
          for (int t = 0; t < m; ++t) {
            // box 1 holds e1: its incoming datum is slot 1; box 2's is slot 0.
            const int in1 = f * bs + m + t, in2 = f * bs + t;
            const int q1 = pos_of[in1], q2 = pos_of[in2];
            if (q1 < 0 || q2 < 0 || bx[0]->pos[q1].in != in1 || bx[1]->pos[q2].in != in2)
              throw std::logic_error("build_hierarchy: separator node not on the merging boxes");
            sep[0].push_back(q1), sep[1].push_back(q2);
            is_sep[0][q1] = 1, is_sep[1][q2] = 1;
          }
        }
        for (int k = 0; k < 2; ++k) {
          std::vector<int>& perm = gp.perm[k];
          for (int i = 0; i < static_cast<int>(bx[k]->pos.size()); ++i)
            if (bx[k]->pos[i].in >= 0 && !is_sep[k][i]) perm.push_back(i);
          gp.p[k] = static_cast<int>(perm.size());
          for (int i : perm) gp.next_pos.push_back(bx[k]->pos[i]);
          if (!gp.own) continue;
          perm.insert(perm.end(), sep[k].begin(), sep[k].end());
          gp.cpos[k].reserve(perm.size());
          for (int i : perm) gp.cpos[k].push_back(bx[k]->pos[i]);
        }
        for (int k = 0; k < 2; ++k)
          for (const auto& q : bx[k]->pos)
            if (q.in >= 0) pos_of[q.in] = -1;
      }
    });
    // serial pass: indices and offsets in group order
    for (int gi = 0; gi < ng; ++gi) {
      GroupPlan& gp = plan[gi];
      next_pos[gi] = std::move(gp.next_pos);
      if (!gp.own) continue;
      const Face& f0 = g.faces[groups[gi][0]];
      const HostBox* bx[2] = {&boxes[elem_box[f0.e1]], &boxes[elem_box[f0.e2]]};
      MergeRec mr;
      mr.s = static_cast<int>(groups[gi].size()) * m;
      mr.group = gi;
      if (level > 1) {
        mr.src1 = prev_merge_of[elem_box[f0.e1]];
        mr.src2 = prev_merge_of[elem_box[f0.e2]];
      }
      for (int k = 0; k < 2; ++k) {
        ChildBox cb;
        cb.p = gp.p[k];
        cb.s = mr.s;
        cb.P = static_cast<int>(gp.perm[k].size());
        cb.pos = std::move(gp.cpos[k]);
        cb.t_off = toff;
        toff += static_cast<size_t>(cb.P) * cb.P;
        (k == 0 ? mr.c1 : mr.c2) = static_cast<int>(L->children.size());
        (k == 0 ? mr.p1 : mr.p2) = cb.p;
        L->children.push_back(std::move(cb));
        perms.push_back(std::move(gp.perm[k]));
        srcs.push_back(bx[k]);
      }
      merge_of[gi] = static_cast<int>(L->merges.size());
      L->merges.push_back(mr);
    }
    tr.mark("bookkeeping");
    prev_merge_of = merge_of;
    L->tperm.alloc(toff);
    tr.mark("alloc");

    // ---- sharded global levels: bring the child maps this rank merges
    // (owner-computes: the second child from its holder, NCCL send / recv),
    // or every child to every rank at the replicated coarse level
    std::vector<DevBuf<double2>> remote;
    if (sharded && level > part.last_local) {
      std::vector<Comm::Xfer> sends, recvs;
      for (int gi = 0; gi < ng; ++gi) {
        const Face& f0 = g.faces[groups[gi][0]];
        const int b1 = elem_box[f0.e1], b2 = elem_box[f0.e2];
        for (const int b : {b1, b2}) {
          HostBox& hb = boxes[b];
          const size_t bytes = sizeof(double2) * static_cast<size_t>(hb.ld) * hb.ld;
          const int holder = box_owner[b];
          if (level == depth) {  // coarse: every box to every rank (broadcast)
            if (holder != me) {
              remote.emplace_back(static_cast<size_t>(hb.ld) * hb.ld);
              hb.T = remote.back().p;
            }
            ctx->comm->broadcast(const_cast<double2*>(hb.T), bytes, holder, ctx);
          } else {
            const int owner = box_owner[b1];
            if (holder == owner) continue;
            if (holder == me) sends.push_back({owner, const_cast<double2*>(hb.T), bytes});
            if (owner == me) {
              remote.emplace_back(static_cast<size_t>(hb.ld) * hb.ld);
              hb.T = remote.back().p;
              recvs.push_back({holder, remote.back().p, bytes});
            }
          }
        }
      }
      if (level < depth) ctx->comm->exchange(sends, recvs, ctx);
      tr.mark("box_exchange");
    }

    // ---- gather children into the permuted layout
    {
      std::vector<int> hperm;
      std::vector<size_t> poff;
      for (const auto& p : perms) {
        poff.push_back(hperm.size());
        hperm.insert(hperm.end(), p.begin(), p.end());
      }
      DevBuf<int> dperm;
      dperm.upload(hperm, ctx->stream);
      CopyBatch cb;
      for (size_t c = 0; c < perms.size(); ++c) {
        const ChildBox& ch = L->children[c];
        cb.gather(srcs[c]->T, srcs[c]->ld, dperm.p + poff[c], dperm.p + poff[c],
                  L->tperm.p + ch.t_off, ch.P, ch.P, ch.P);
      }
      cb.run(ctx);
      tr.mark("gather_enqueue");
      // No synchronisation: buffers are freed stream-ordered, so the host
      // moves on to the next level's bookkeeping while the GPU works.
    }
    tnew_prev.release();

    // ---- V-cycle / export index lists (offsets serially, fill in parallel)
    {
      size_t total_idx = 0;
      for (auto& mr : L->merges) {
        const ChildBox& a = L->children[mr.c1];
        const ChildBox& b = L->children[mr.c2];
        mr.in1_sep = total_idx, total_idx += a.P - a.p;
        mr.in2_sep = total_idx, total_idx += b.P - b.p;
        mr.in1_per = total_idx, total_idx += a.p;
        mr.out1_per = total_idx, total_idx += a.p;
        mr.in2_per = total_idx, total_idx += b.p;
        mr.out2_per = total_idx, total_idx += b.p;
      }
      L->h_idx.resize(total_idx);
      parallel_chunks(static_cast<int>(L->merges.size()), host_threads(), [&](int m0, int m1, int) {
        for (int gi = m0; gi < m1; ++gi) {
          const MergeRec& mr = L->merges[gi];
          const ChildBox& a = L->children[mr.c1];
          const ChildBox& b = L->children[mr.c2];
          auto put = [&](const ChildBox& c, int from, int to, bool in, size_t at) {
            for (int i = from; i < to; ++i) L->h_idx[at++] = in ? c.pos[i].in : c.pos[i].out;
          };
          put(a, a.p, a.P, true, mr.in1_sep);
          put(b, b.p, b.P, true, mr.in2_sep);
          put(a, 0, a.p, true, mr.in1_per);
          put(a, 0, a.p, false, mr.out1_per);
          put(b, 0, b.p, true, mr.in2_per);
          put(b, 0, b.p, false, mr.out2_per);
        }
      });
    }

    if (!L->coarse) {
      // ---- merges (this rank's)
      const int nm = static_cast<int>(L->merges.size());
      size_t woff = 0, roff = 0, noff = 0;
      std::vector<size_t> r_at(nm), n_at(nm);
      for (int gi = 0; gi < nm; ++gi) {
        MergeRec& mr = L->merges[gi];
        const int q = mr.p1 + mr.p2;
        mr.w_off = woff;
        woff += static_cast<size_t>(mr.s) * mr.s;
        r_at[gi] = roff;
        roff += static_cast<size_t>(mr.s) * q;
        n_at[gi] = noff;
        noff += static_cast<size_t>(q) * q;
      }
      L->w.alloc(woff);
      tr.mark("idx");
      DevBuf<double2> R(roff), X1(roff), X2(roff), tnew(noff);
      tr.mark("alloc");
      CopyBatch pre;
      GemmBatch g1, g2, g3, g4;
      InverseBatch inv;
      for (int gi = 0; gi < nm; ++gi) {
        const MergeRec& mr = L->merges[gi];
        const ChildBox& c1 = L->children[mr.c1];
        const ChildBox& c2 = L->children[mr.c2];
        const int s = mr.s, p1 = mr.p1, p2 = mr.p2, q = p1 + p2, P1 = c1.P, P2 = c2.P;
        const double2* T1 = L->tperm.p + c1.t_off;
        const double2* T2 = L->tperm.p + c2.t_off;
        const double2 *T1pp = T1, *T1ps = T1 + static_cast<size_t>(p1) * P1, *T1sp = T1 + p1,
                      *T1ss = T1 + p1 + static_cast<size_t>(p1) * P1;
        const double2 *T2pp = T2, *T2ps = T2 + static_cast<size_t>(p2) * P2, *T2sp = T2 + p2,
                      *T2ss = T2 + p2 + static_cast<size_t>(p2) * P2;
        double2* W = L->w.p + mr.w_off;
        double2* Rg = R.p + r_at[gi];
        double2* X1g = X1.p + r_at[gi];
        double2* X2g = X2.p + r_at[gi];
        double2* Tn = tnew.p + n_at[gi];
        // X2 and T_new are write-only outputs: their additive terms are read
        // from the child blocks where they lie (GemmDesc::Cin), not staged.
        pre.identity(W, s, s);
        pre.copy(T2sp, P2, Rg + static_cast<size_t>(p1) * s, s, s, p2, -1.0);
        g1.add(T2ss, P2, T1ss, P1, W, s, s, s, s, -1.0, 1.0);
        g1.add(T2ss, P2, T1sp, P1, Rg, s, s, p1, s, 1.0, 0.0);
        inv.ops.push_back(InvOp{W, s, s, (level << 20) | mr.group, 0});
        g2.add(W, s, Rg, s, X1g, s, s, q, s, 1.0, 0.0);  // X1 = W [T2_ss T1_sp, -T2_sp]
        {  // X2 = -T1_ss X1 - [T1_sp, 0]
          GemmDesc d{};
          d.A = T1ss, d.lda = P1, d.B = X1g, d.ldb = s, d.C = X2g, d.ldc = s, d.M = s, d.N = q, d.K = s;
          d.alpha_re = -1.0, d.beta_re = -1.0, d.Cin = T1sp, d.ldcin = P1, d.cin_c0 = 0, d.cin_c1 = p1;
          g3.add(d);
        }
        {  // T_new[0:p1, :] = [T1_pp, 0] + T1_ps X1
          GemmDesc d{};
          d.A = T1ps, d.lda = P1, d.B = X1g, d.ldb = s, d.C = Tn, d.ldc = q, d.M = p1, d.N = q, d.K = s;
          d.alpha_re = 1.0, d.beta_re = 1.0, d.Cin = T1pp, d.ldcin = P1, d.cin_c0 = 0, d.cin_c1 = p1;
          g3.add(d);
        }
        {  // T_new[p1:q, :] = [0, T2_pp] + T2_ps X2
          GemmDesc d{};
          d.A = T2ps, d.lda = P2, d.B = X2g, d.ldb = s, d.C = Tn + p1, d.ldc = q, d.M = p2, d.N = q, d.K = s;
          d.alpha_re = 1.0, d.beta_re = 1.0, d.Cin = T2pp, d.ldcin = P2, d.cin_c0 = p1, d.cin_c1 = q;
          g4.add(d);
        }
      }
      tr.mark("merge_lists");
      pre.run(ctx);
      g1.run(ctx);
      tr.mark("merge_run_g1");
      inv.diag_pivots = !pivot;
      inv.guard_dev = d_status.p + 1;
      inv.run(ctx, d_status.p);
      tr.mark("merge_run_inv");
      g2.run(ctx);
      g3.run(ctx);
      g4.run(ctx);
      L->merge_flops = g1.flops + g2.flops + g3.flops + g4.flops;
      for (const auto& mr : L->merges) L->merge_flops += 8.0 * mr.s * mr.s * mr.s;  // inverse
      tr.mark("merge_enqueue");
      // ---- next level's boxes (positions for every group, maps for ours)
      std::vector<HostBox> next(ng);
      for (int gi = 0; gi < ng; ++gi) {
        HostBox& nbx = next[gi];
        nbx.pos = std::move(next_pos[gi]);
        nbx.ld = static_cast<int>(nbx.pos.size());
        nbx.T = merge_of[gi] >= 0 ? tnew.p + n_at[merge_of[gi]] : nullptr;
      }
      box_owner = sharded ? owners[level - 1] : std::vector<int>(ng, 0);
      // element -> new box: the merge owning the element's old box
      std::vector<int> box_to_group(boxes.size(), -1);
      for (int gi = 0; gi < ng; ++gi) {
        const Face& f0 = g.faces[groups[gi][0]];
        box_to_group[elem_box[f0.e1]] = gi;
        box_to_group[elem_box[f0.e2]] = gi;
      }
      for (int e = 0; e < ne; ++e) elem_box[e] = box_to_group[elem_box[e]];
      boxes = std::move(next);
      tnew_prev = std::move(tnew);
    }
    L->idx.upload(L->h_idx, ctx->stream);
    h->device_bytes += static_cast<int64_t>(L->tperm.bytes() + L->w.bytes() + L->idx.bytes());
    h->levels.push_back(std::move(L));
  }
  HPSB_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  // status into pinned memory: a copy to pageable memory would block the host
  // until the stream drains (before the hook could overlap it)
  thread_local int* st_pinned = [] {
    int* q = nullptr;
    HPSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&q), 2 * sizeof(int)));
    return q;
  }();
  st_pinned[0] = st_pinned[1] = 0;
  HPSB_CUDA(cudaMemcpyAsync(st_pinned, d_status.p, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream));
  if (before_wait) {
    // the hook's own device work is stream-ordered after the merges: record
    // the build's end event first (above), so build_seconds stays the merges'
    before_wait(h.get());
    tr.mark("before_wait_hook");
  }
  HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
  tr.mark("final_wait");
  elements_wait(sk->el);  // long finished: the merges consumed the element maps
  int st = st_pinned[0];
  bool trip = st_pinned[1] != 0 || (!pivot && std::getenv("HPSB_TEST_GUARD_TRIP"));
  if (sharded) {
    // test hook: trip the guard on one rank only
    if (const char* r = std::getenv("HPSB_TEST_GUARD_TRIP_RANK"))
      trip |= !pivot && std::atoi(r) == ctx->rank();
    // The guard and the singular-block status are per rank (each rank merged
    // its own subtree): agree on them, so that every rank redoes the build
    // (and its collectives) together, or every rank throws.
    DevBuf<double2> flag(1);
    const double2 mine = make_double2(trip ? 1.0 : 0.0, st ? 1.0 : 0.0);
    HPSB_CUDA(cudaMemcpyAsync(flag.p, &mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream));
    ctx->comm->allreduce_sum(flag.p, 1, ctx);
    double2 all;
    HPSB_CUDA(cudaMemcpyAsync(&all, flag.p, sizeof(all), cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    trip = all.x > 0.0;
    if (!st && all.y > 0.0)
      throw std::runtime_error("eliminate_level: singular merge block on another rank");
  }
  *guard_tripped = trip;
  if (*guard_tripped) return h;  // results unused: the caller redoes the build
  if (st) {  // first singular group pivot (inverse status tag = level << 20 | group) + 1
    const int tag = st - 1, level = tag >> 20, gi = tag & ((1 << 20) - 1);
    throw std::runtime_error("eliminate_level: singular merge block at face " +
                             std::to_string(g.groups[level - 1][gi].front()));
  }
  float ms = 0;
  HPSB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
  h->build_seconds = ms * 1e-3;
  return h;
}

std::unique_ptr<Hierarchy> build_hierarchy(Skeleton* sk, int depth,
                                           const std::function<void(Hierarchy*)>& before_wait) {
  const bool pivot = std::getenv("HPSB_MERGE_PIVOT") != nullptr;
  bool tripped = false;
  auto h = build_hierarchy_pass(sk, depth, before_wait, pivot, &tripped);
  if (!tripped) return h;
  h.reset();
  h = build_hierarchy_pass(sk, depth, before_wait, true, &tripped);
  h->pivot_redone = true;
  return h;
}

void hierarchy_pinned(const Hierarchy* h, double* elem_flops, double* merge_flops,
                      double* level_entries) {
  const Elements* el = h->sk->el;
  const double ni = static_cast<double>(el->m) * el->m, nb = el->nb;
  const double ne = static_cast<double>(el->n) * el->n;
  if (elem_flops) *elem_flops = ne * (ni * ni * ni / 3.0 + 2.0 * ni * ni * nb + 8.0 * nb * nb * nb);
  double fm = 0, ent = 0;
  for (const auto& L : h->levels) {
    if (L->coarse) continue;
    for (const MergeRec& mr : L->merges) {
      const double s = mr.s, p = mr.p1 + mr.p2;
      fm += 8.0 * ((8.0 / 3.0) * s * s * s + 4.0 * s * s * p + s * p * p);
      ent += 2.0 * (2.0 * s) * (2.0 * s) + 2.0 * s * p;
    }
  }
  if (merge_flops) *merge_flops = fm;
  if (level_entries) *level_entries = ent;
}

// M_l in the reference's bs x bs block layout (for parity tests / export).
void hierarchy_level_blocks(const Hierarchy* h, int level, int* nblocks, int* first_face,
                            int* keys, double* data) {
  if (level < 1 || level > h->depth) throw InvalidArgument("level out of range");
  const LevelOps& L = *h->levels[level - 1];
  const int bs = h->sk->bs, ff = L.first_face;
  std::unordered_map<int64_t, std::vector<double2>> blocks;
  auto key_of = [&](int r, int c) { return static_cast<int64_t>(r) * L.nfaces + c; };
  auto blk = [&](int r, int c) -> std::vector<double2>& {
    auto& b = blocks[key_of(r, c)];
    if (b.empty()) b.assign(static_cast<size_t>(bs) * bs, make_double2(0.0, 0.0));
    return b;
  };
  for (int f = 0; f < L.nfaces; ++f) {
    auto& b = blk(f, f);
    for (int k = 0; k < bs; ++k) b[k + k * bs].x += 1.0;
  }
  std::vector<double2> T;
  for (const ChildBox& c : L.children) {
    T.resize(static_cast<size_t>(c.P) * c.P);
    HPSB_CUDA(cudaMemcpy(T.data(), L.tperm.p + c.t_off, T.size() * sizeof(double2),
                         cudaMemcpyDeviceToHost));
    for (int j = 0; j < c.P; ++j)
      for (int i = 0; i < c.P; ++i) {
        const int row = c.pos[i].out, col = c.pos[j].in;
        auto& b = blk(row / bs - ff, col / bs - ff);
        double2& v = b[(row % bs) + static_cast<size_t>(col % bs) * bs];
        const double2 t = T[i + static_cast<size_t>(j) * c.P];
        v.x += t.x, v.y += t.y;
      }
  }
  *first_face = ff;
  if (!keys) {
    *nblocks = static_cast<int>(blocks.size());
    return;
  }
  std::vector<int64_t> order;
  for (const auto& kv : blocks) order.push_back(kv.first);
  std::sort(order.begin(), order.end());
  int k = 0;
  for (int64_t key : order) {
    keys[2 * k] = static_cast<int>(key / L.nfaces);
    keys[2 * k + 1] = static_cast<int>(key % L.nfaces);
    std::memcpy(data + 2 * static_cast<size_t>(k) * bs * bs, blocks[key].data(),
                sizeof(double2) * bs * bs);
    ++k;
  }
  *nblocks = k;
}

}  // namespace hpsb

namespace hpsb {

// merge_pair (proj/src/dissection.cpp:23-82): the same box merge on two
// elements, fused layout [e1 sides minus alpha | e2 sides minus beta] in
// left/right/bottom/top order, plus the source term
//   H_pair = [H1_p + T1_ps x1; H2_p + T2_ps x2],
//   x1 = W (T2_ss H1_s - H2_s),  x2 = -H1_s - T1_ss x1.
void merge_pair(Context* ctx, int m, const double2* T1h, const double2* H1h, const double2* T2h,
                const double2* H2h, int alpha, int beta, double2* Th, double2* Hh) {
  const int nb = 4 * m, s = m, p = 3 * m, q = 6 * m;
  std::vector<int> perm;
  for (int k = 0; k < 2; ++k) {
    const int skip = k == 0 ? alpha : beta;
    for (int side = 0; side < 4; ++side)
      if (side != skip)
        for (int t = 0; t < m; ++t) perm.push_back(side * m + t);
    for (int t = 0; t < m; ++t) perm.push_back(skip * m + t);
  }
  DevBuf<int> dperm;
  dperm.upload(perm, ctx->stream);
  DevBuf<double2> T1(nb * nb), T2(nb * nb), H1(nb), H2(nb), P1(nb * nb), P2(nb * nb), h1(nb),
      h2(nb), W(s * s), R(s * q), X1(s * q), X2(s * q), Tn(q * q), u(s), x1(s), x2(s), Hn(q);
  HPSB_CUDA(cudaMemcpyAsync(T1.p, T1h, T1.bytes(), cudaMemcpyHostToDevice, ctx->stream));
  HPSB_CUDA(cudaMemcpyAsync(T2.p, T2h, T2.bytes(), cudaMemcpyHostToDevice, ctx->stream));
  HPSB_CUDA(cudaMemcpyAsync(H1.p, H1h, H1.bytes(), cudaMemcpyHostToDevice, ctx->stream));
  HPSB_CUDA(cudaMemcpyAsync(H2.p, H2h, H2.bytes(), cudaMemcpyHostToDevice, ctx->stream));
  CopyBatch gat;
  gat.gather(T1.p, nb, dperm.p, dperm.p, P1.p, nb, nb, nb);
  gat.gather(T2.p, nb, dperm.p + nb, dperm.p + nb, P2.p, nb, nb, nb);
  gat.gather(H1.p, nb, dperm.p, nullptr, h1.p, nb, nb, 1);
  gat.gather(H2.p, nb, dperm.p + nb, nullptr, h2.p, nb, nb, 1);
  gat.run(ctx);
  HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
  const double2 *T1pp = P1.p, *T1ps = P1.p + p * nb, *T1sp = P1.p + p, *T1ss = P1.p + p + p * nb;
  const double2 *T2pp = P2.p, *T2ps = P2.p + p * nb, *T2sp = P2.p + p, *T2ss = P2.p + p + p * nb;
  CopyBatch pre;
  pre.identity(W.p, s, s);
  pre.copy(T2sp, nb, R.p + p * s, s, s, p, -1.0);
  pre.copy(T1sp, nb, X2.p, s, s, p, -1.0);
  pre.zero(X2.p + p * s, s, s, p);
  pre.copy(T1pp, nb, Tn.p, q, p, p, 1.0);
  pre.zero(Tn.p + p * q, q, p, p);
  pre.zero(Tn.p + p, q, p, p);
  pre.copy(T2pp, nb, Tn.p + p + p * q, q, p, p, 1.0);
  pre.copy(h2.p + p, nb, u.p, s, s, 1, -1.0);
  pre.copy(h1.p + p, nb, x2.p, s, s, 1, -1.0);
  pre.copy(h1.p, nb, Hn.p, q, p, 1, 1.0);
  pre.copy(h2.p, nb, Hn.p + p, q, p, 1, 1.0);
  pre.run(ctx);
  GemmBatch g1, g2, g3, g4;
  g1.add(T2ss, nb, T1ss, nb, W.p, s, s, s, s, -1.0, 1.0);
  g1.add(T2ss, nb, T1sp, nb, R.p, s, s, p, s, 1.0, 0.0);
  g1.add(T2ss, nb, h1.p + p, nb, u.p, s, s, 1, s, 1.0, 1.0);
  g1.run(ctx);
  DevBuf<int> st(1);
  HPSB_CUDA(cudaMemsetAsync(st.p, 0, sizeof(int), ctx->stream));
  InverseBatch inv;
  inv.ops.push_back(InvOp{W.p, s, s, 0, 0});
  inv.run(ctx, st.p);
  g2.add(W.p, s, R.p, s, X1.p, s, s, q, s, 1.0, 0.0);
  g2.add(W.p, s, u.p, s, x1.p, s, s, 1, s, 1.0, 0.0);
  g2.run(ctx);
  g3.add(T1ss, nb, X1.p, s, X2.p, s, s, q, s, -1.0, 1.0);
  g3.add(T1ps, nb, X1.p, s, Tn.p, q, p, q, s, 1.0, 1.0);
  g3.add(T1ss, nb, x1.p, s, x2.p, s, s, 1, s, -1.0, 1.0);
  g3.add(T1ps, nb, x1.p, s, Hn.p, q, p, 1, s, 1.0, 1.0);
  g3.run(ctx);
  g4.add(T2ps, nb, X2.p, s, Tn.p + p, q, p, q, s, 1.0, 1.0);
  g4.add(T2ps, nb, x2.p, s, Hn.p + p, q, p, 1, s, 1.0, 1.0);
  g4.run(ctx);
  int fail = 0;
  HPSB_CUDA(cudaMemcpyAsync(&fail, st.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  HPSB_CUDA(cudaMemcpyAsync(Th, Tn.p, Tn.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
  HPSB_CUDA(cudaMemcpyAsync(Hh, Hn.p, Hn.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
  HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (fail) throw std::runtime_error("merge_pair: singular face block");
}

}  // namespace hpsb
