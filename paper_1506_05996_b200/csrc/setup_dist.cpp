// Element-slab partition of the solve for the distributed plan.
// Host-only C++: every rank runs the same deterministic setup on the full
// mesh and keeps the parts it needs, so both sides of every exchange derive
// identical lists without talking.
//
// Ranks own contiguous element ranges [r*NE/R, (r+1)*NE/R). A node is
// finalised by the rank of its highest-numbered copy's element (interior
// nodes by their element's rank): the Ax continuation of kernels_gather.cuh
// (lower rank's copies first) ends there, and so does every other sum over
// the node's contributions, which are all kept in the reference order.
#include <algorithm>
#include <cstring>

#include "../../include/hexsem_b200.h"
#include "setup.hpp"

namespace hxb {

namespace {
int slab_start(int ne, int r, int R) { return static_cast<int>(static_cast<long long>(ne) * r / R); }
int slab_of(int ne, int e, int R)
{
  int r = static_cast<int>((static_cast<long long>(e) * R) / ne);
  while (r > 0 && e < slab_start(ne, r, R)) --r;
  while (r + 1 < R && e >= slab_start(ne, r + 1, R)) ++r;
  return r;
}
}  // namespace

DistLists dist_partition(const HostSetup& hs, int rank, int nranks, int nsurfp)
{
  const Numbering& num = hs.num;
  const int ne_all = hs.mesh.num_elements();
  const int np = hs.order + 1;
  const int nsurf_raw = surface_slot_count(np);
  auto start = [&](int r) { return static_cast<int>(static_cast<long long>(ne_all) * r / nranks); };
  const int e0 = start(rank), e1 = start(rank + 1);
  const int e_lo = rank > 0 ? start(rank - 1) : 0, e_hi = rank + 1 < nranks ? start(rank + 2) : ne_all;
  const int nsg = num.num_surface_global;
  std::vector<int> minE(nsg, ne_all), maxE(nsg, -1);
  for (int e = 0; e < ne_all; ++e)
    for (int q = 0; q < nsurf_raw; ++q) {
      const gid g = num.l2g_surf[static_cast<std::size_t>(e) * nsurf_raw + q];
      minE[g] = std::min(minE[g], e);
      maxE[g] = std::max(maxE[g], e);
    }
  std::vector<int> loc(nsg, -1);
  std::vector<gid> grp[3];
  for (int e = e0; e < e1; ++e)
    for (int q = 0; q < nsurf_raw; ++q) {
      const gid g = num.l2g_surf[static_cast<std::size_t>(e) * nsurf_raw + q];
      if (loc[g] != -1) continue;
      loc[g] = -2;
      const bool up = maxE[g] >= e1, down = minE[g] < e0;
      if ((up && down) || (up && maxE[g] >= e_hi) || (down && minE[g] < e_lo))
        throw HxbError(HXB_EINVAL, "slab partition too thin: a node spans more than two ranks");
      grp[up ? 1 : (down ? 2 : 0)].push_back(g);
    }
  DistLists d;
  d.e0 = e0;
  d.e1 = e1;
  for (auto& v : grp) {
    std::sort(v.begin(), v.end());
    d.nodes.insert(d.nodes.end(), v.begin(), v.end());
  }
  d.n_grp0 = static_cast<int>(grp[0].size());
  d.n_up = static_cast<int>(grp[1].size());
  d.n_down = static_cast<int>(grp[2].size());
  const int nl = static_cast<int>(d.nodes.size());
  for (int t = 0; t < nl; ++t) loc[d.nodes[t]] = t;
  d.off.assign(static_cast<std::size_t>(nl) + 1, 0);
  for (int e = e0; e < e1; ++e)
    for (int q = 0; q < nsurf_raw; ++q) d.off[loc[num.l2g_surf[static_cast<std::size_t>(e) * nsurf_raw + q]] + 1]++;
  for (int t = 0; t < nl; ++t) d.off[t + 1] += d.off[t];
  std::vector<unsigned> cur(d.off.begin(), d.off.end() - 1);
  d.smap.assign(static_cast<std::size_t>(e1 - e0) * 2 * nsurfp, 0);
  d.idx.assign(d.off[nl], 0);
  for (int le = 0; le < e1 - e0; ++le)
    for (int q = 0; q < nsurf_raw; ++q) {
      const gid g = num.l2g_surf[static_cast<std::size_t>(e0 + le) * nsurf_raw + q];
      int* row = &d.smap[static_cast<std::size_t>(le) * 2 * nsurfp];
      row[q] = num.dirichlet_mask[g] ? -g - 2 : g;  // encode_dirichlet
      const unsigned pos = cur[loc[g]]++;
      row[nsurfp + q] = static_cast<int>(pos);
      d.idx[pos] = le * nsurfp + q;
    }
  return d;
}



DistPcgLists dist_pcg_setup(const HostSetup& hs, const DistLists& d, int rank, int nranks)
{
  const Numbering& num = hs.num;
  const int ne = hs.mesh.num_elements();
  const int n = hs.order, np = n + 1, P = n + 3, nloc = np * np * np, nsub = P * P * P;
  const int nsurf_raw = surface_slot_count(np);
  const gid nsg = num.num_surface_global, N = num.num_global;
  const std::int64_t NI = static_cast<std::int64_t>(n - 1) * (n - 1) * (n - 1);
  const int e0 = d.e0, e1 = d.e1;
  DistPcgLists o;
  // finaliser of every node
  std::vector<int> maxE(nsg, -1);
  for (int e = 0; e < ne; ++e)
    for (int q = 0; q < nsurf_raw; ++q) {
      const gid g = num.l2g_surf[static_cast<std::size_t>(e) * nsurf_raw + q];
      maxE[g] = std::max(maxE[g], e);
    }
  auto fin = [&](gid g) {
    const int e = g < nsg ? maxE[g] : static_cast<int>((g - nsg) / NI);
    return slab_of(ne, e, nranks);
  };
  // local nodes of this rank (surface list + interior range)
  std::vector<char> local(N, 0);
  for (gid g : d.nodes) local[g] = 1;
  const gid ib0 = static_cast<gid>(nsg + e0 * NI), ib1 = static_cast<gid>(nsg + e1 * NI);
  for (gid g = ib0; g < ib1; ++g) local[g] = 1;
  o.ib0 = ib0;
  o.ib1 = ib1;
  // finalised surface nodes (group 0 + down) in the order of the local list
  for (int t = 0; t < d.n_grp0; ++t) o.fin_surf.push_back(d.nodes[t]);
  for (int t = d.n_grp0 + d.n_up; t < static_cast<int>(d.nodes.size()); ++t) o.fin_surf.push_back(d.nodes[t]);
  // position of every finalised node in the combine's item order
  std::vector<int> item(N, -1);
  for (std::size_t t = 0; t < o.fin_surf.size(); ++t) item[o.fin_surf[t]] = static_cast<int>(t);
  const int nfs = static_cast<int>(o.fin_surf.size());
  for (gid g = ib0; g < ib1; ++g) item[g] = nfs + (g - ib0);
  const int nitems = nfs + (ib1 - ib0);
  // fine contributions of every finalised node, in (e, slot) order
  std::vector<gid> scratch(nloc);
  o.fine_off.assign(static_cast<std::size_t>(nitems) + 1, 0);
  // only elements whose subdomain can touch this rank's finalised nodes: the
  // owned slab and one element layer either side is not enough for thin
  // slabs, so scan the neighbour slabs entirely
  const int s_lo = rank > 0 ? slab_start(ne, rank - 1, nranks) : 0;
  const int s_hi = rank + 1 < nranks ? slab_start(ne, rank + 2, nranks) : ne;
  for (int e = s_lo; e < s_hi; ++e)
    for_each_sub_slot(num, ne, e, scratch.data(), [&](gid g, int) {
      if (g >= 0 && item[g] >= 0) o.fine_off[item[g] + 1]++;
    });
  for (int t = 0; t < nitems; ++t) o.fine_off[t + 1] += o.fine_off[t];
  std::vector<unsigned> cur(o.fine_off.begin(), o.fine_off.end() - 1);
  o.fine_pos.assign(static_cast<std::size_t>(e1 - e0) * nsub, -1);
  int nto[2] = {0, 0};  // contributions this rank sends down / up
  for (int e = s_lo; e < s_hi; ++e) {
    const int re = slab_of(ne, e, nranks);
    for_each_sub_slot(num, ne, e, scratch.data(), [&](gid g, int slot) {
      if (g < 0) return;
      const int fr = fin(g);
      if (item[g] >= 0) {  // finalised here: a local sum position
        const unsigned pos = cur[item[g]]++;
        if (re == rank) {
          o.fine_pos[static_cast<std::size_t>(e - e0) * nsub + slot] = static_cast<int>(pos);
        } else {  // computed by neighbour re, received into pos
          if (re != rank - 1 && re != rank + 1) throw HxbError(1, "slab partition too thin for the fine halo");
          (re < rank ? o.frecv_down : o.frecv_up).push_back(static_cast<int>(pos));
        }
      } else if (re == rank) {  // computed here, finalised by a neighbour: send
        if (fr != rank - 1 && fr != rank + 1) throw HxbError(1, "slab partition too thin for the fine halo");
        const int side = fr < rank ? 0 : 1;
        o.fine_pos[static_cast<std::size_t>(e - e0) * nsub + slot] = -2 - (side ? (1 << 30) + nto[1] : nto[0]);
        ++nto[side];
      }
    });
  }
  o.n_fsend_down = nto[0];
  o.n_fsend_up = nto[1];
  // pack codes into one send buffer [down | up]
  for (int& q : o.fine_pos)
    if (q <= -2) {
      const int c = -2 - q;
      q = -2 - (c >= (1 << 30) ? o.n_fsend_down + (c - (1 << 30)) : c);
    }
  // ghost r: sub-slot nodes of owned elements that are not local; the finaliser sends them
  std::vector<gid> gh[2];  // from down / from up
  std::vector<char> seen(N, 0);
  for (int e = e0; e < e1; ++e)
    for_each_sub_slot(num, ne, e, scratch.data(), [&](gid g, int) {
      if (g < 0 || local[g] || seen[g]) return;
      seen[g] = 1;
      const int fr = fin(g);
      if (fr != rank - 1 && fr != rank + 1) throw HxbError(1, "slab partition too thin for the fine halo");
      gh[fr < rank ? 0 : 1].push_back(g);
    });
  for (auto& v : gh) std::sort(v.begin(), v.end());
  o.ghost_from_down = gh[0];
  o.ghost_from_up = gh[1];
  // what the neighbours need from this rank (same rule, evaluated for them)
  for (int side = 0; side < 2; ++side) {
    const int nb = side == 0 ? rank - 1 : rank + 1;
    if (nb < 0 || nb >= nranks) continue;
    const int b0 = slab_start(ne, nb, nranks), b1 = slab_start(ne, nb + 1, nranks);
    std::vector<char> nlocal(N, 0);
    for (int e = b0; e < b1; ++e) {
      element_l2g(num, ne, e, scratch.data());
      for (int l = 0; l < nloc; ++l) nlocal[scratch[l]] = 1;
    }
    std::vector<gid> lst;
    std::vector<char> nseen(N, 0);
    for (int e = b0; e < b1; ++e)
      for_each_sub_slot(num, ne, e, scratch.data(), [&](gid g, int) {
        if (g < 0 || nlocal[g] || nseen[g]) return;
        nseen[g] = 1;
        if (fin(g) == rank) lst.push_back(g);
      });
    std::sort(lst.begin(), lst.end());
    (side == 0 ? o.ghost_to_down : o.ghost_to_up) = lst;
  }
  // coarse prolongation of finalised surface nodes: every copy (e, slot) in
  // (e, l) order with its mass (coarse.cpp:164-186); interior nodes use their element
  const int nsurfp = (nsurf_raw + 3) & ~3;
  std::vector<int> slot_l(nsurf_raw);
  for (int k = 0; k < np; ++k)
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < np; ++i) {
        const int sl = surface_slot_of(np, i, j, k);
        if (sl >= 0) slot_l[sl] = (k * np + j) * np + i;
      }
  o.pr_off.assign(static_cast<std::size_t>(nfs) + 1, 0);
  for (int e = s_lo; e < s_hi; ++e)
    for (int q = 0; q < nsurf_raw; ++q) {
      const gid g = num.l2g_surf[static_cast<std::size_t>(e) * nsurf_raw + q];
      if (item[g] >= 0 && item[g] < nfs) o.pr_off[item[g] + 1]++;
    }
  for (int t = 0; t < nfs; ++t) o.pr_off[t + 1] += o.pr_off[t];
  o.pr_idx.assign(o.pr_off[nfs], 0);
  o.pr_mass.assign(o.pr_off[nfs], 0.0);
  std::vector<unsigned> pc(o.pr_off.begin(), o.pr_off.end() - 1);
  for (int e = s_lo; e < s_hi; ++e)
    for (int q = 0; q < nsurf_raw; ++q) {
      const gid g = num.l2g_surf[static_cast<std::size_t>(e) * nsurf_raw + q];
      if (item[g] < 0 || item[g] >= nfs) continue;
      const unsigned p = pc[item[g]]++;
      o.pr_idx[p] = e * nsurfp + q;
      o.pr_mass[p] = hs.geo.mass[static_cast<std::size_t>(e) * nloc + slot_l[q]];
    }
  return o;
}

// global_node_coords (mesh.cpp:477-492): every element's copy writes its
// trilinear image in (e, l) order, so the last copy wins, as in the reference.
std::vector<double> global_node_coords(const HostSetup& hs)
{
  const Numbering& num = hs.num;
  const int ne = hs.mesh.num_elements();
  const int np = hs.order + 1, nloc = np * np * np;
  std::vector<double> xyz(3 * static_cast<std::size_t>(num.num_global));
  std::vector<gid> l2g(nloc);
  for (int e = 0; e < ne; ++e) {
    element_l2g(num, ne, e, l2g.data());
    int l = 0;
    for (int k = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++l) {
          const auto p = trilinear_map(hs.mesh, e, hs.basis.nodes[i], hs.basis.nodes[j], hs.basis.nodes[k]);
          for (int d = 0; d < 3; ++d) xyz[3 * static_cast<std::size_t>(l2g[l]) + d] = p[d];
        }
  }
  return xyz;
}

}  // namespace hxb
