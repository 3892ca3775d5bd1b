// ingest_text.cu — the text formats of load_mesh, with the reference's
// semantics (mesh_io.cpp):
//   * OBJ (mesh_io.cpp:46-82): "v x y z" and "f i[/..] j k ..." lines; 1-based or negative
//     (relative) indices; polygons fanned by add_polygon (mesh_io.cpp:32-42)
//   * PLY (mesh_io.cpp:137-245) whose body the GPU decoder cannot take as fixed-size records:
//     ASCII bodies and binary bodies with variable face lists, decoded record by record
//   * ASCII STL (mesh_io.cpp:320-342): "vertex x y z" triples; corners welded on the GPU by exact
//     double equality in first-occurrence order (the binary path's weld, on 64-bit keys)
// Text is tokenised on the host (std::from_chars: correctly rounded doubles, as the reference's
// istream extraction); the corner weld, degenerate-face drop and device upload run on the GPU.
// Parse errors are PAMOPT_CU_EIO with the reference's message (std::runtime_error there).
#include <cub/cub.cuh>

#include <charconv>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

[[noreturn]] void fail(const std::string& what, long line = -1) {
  std::string msg = what;
  if (line >= 0) msg += " (line " + std::to_string(line) + ")";
  throw Error(PAMOPT_CU_EIO, msg);
}

// whitespace tokenizer over one line (istringstream >> semantics for the token boundaries)
struct Tokens {
  std::string_view s;
  size_t p = 0;
  bool next(std::string_view& t) {
    while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
    if (p >= s.size()) return false;
    const size_t b = p;
    while (p < s.size() && !std::isspace(static_cast<unsigned char>(s[p]))) ++p;
    t = s.substr(b, p - b);
    return true;
  }
};

// istream >> double on a whitespace token: optional sign, decimal digits, point, exponent;
// correctly rounded (from_chars); no inf / nan / hex (num_get's grammar has none)
bool to_double(std::string_view t, double& v) {
  if (!t.empty() && t[0] == '+') t.remove_prefix(1);
  if (t.empty()) return false;
  for (char c : t)
    if (!(std::isdigit(static_cast<unsigned char>(c)) || c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+'))
      return false;
  auto r = std::from_chars(t.data(), t.data() + t.size(), v, std::chars_format::general);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
template <class I>
bool to_int(std::string_view t, I& v) {
  if (!t.empty() && t[0] == '+') t.remove_prefix(1);
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}

struct HostMesh {
  std::vector<double> V;
  std::vector<int32_t> F;
  int64_t triangulated = 0, degenerate = 0;
  int64_t nv() const { return static_cast<int64_t>(V.size() / 3); }
  // add_polygon (mesh_io.cpp:32-42): fan from the first vertex, repeated-index triangles dropped
  void add_polygon(const std::vector<int64_t>& poly) {
    if (poly.size() > 3) ++triangulated;
    for (size_t k = 1; k + 1 < poly.size(); ++k) {
      const int64_t a = poly[0], b = poly[k], c = poly[k + 1];
      if (a == b || b == c || a == c) {
        ++degenerate;
        continue;
      }
      F.push_back(static_cast<int32_t>(a));
      F.push_back(static_cast<int32_t>(b));
      F.push_back(static_cast<int32_t>(c));
    }
  }
};

void upload(Ctx& ctx, const HostMesh& h, IngestResult& out) {
  out = IngestResult();
  out.nv = h.nv();
  out.nf = static_cast<int64_t>(h.F.size() / 3);
  out.degenerate_dropped = h.degenerate;
  out.V.alloc(h.V.empty() ? 1 : h.V.size(), ctx.stream);
  out.F.alloc(h.F.empty() ? 1 : h.F.size(), ctx.stream);
  if (!h.V.empty())
    PCU_CUDA(cudaMemcpyAsync(out.V.get(), h.V.data(), h.V.size() * 8, cudaMemcpyHostToDevice, ctx.stream));
  if (!h.F.empty())
    PCU_CUDA(cudaMemcpyAsync(out.F.get(), h.F.data(), h.F.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));  // the host vectors die with the caller
}

// lines of a buffer (getline semantics; a trailing '\r' is kept for OBJ as the reference does,
// where it only ends a token)
template <class Fn>
void for_lines(const char* b, int64_t n, Fn&& fn) {
  long lineno = 0;
  int64_t p = 0;
  while (p < n) {
    int64_t e = p;
    while (e < n && b[e] != '\n') ++e;
    ++lineno;
    fn(std::string_view(b + p, static_cast<size_t>(e - p)), lineno);
    p = e + 1;
  }
}

// ------------------------------------------------------------------- double-corner weld (GPU)
__device__ __forceinline__ bool isnan64(uint64_t b) {
  return (b & 0x7ff0000000000000ull) == 0x7ff0000000000000ull && (b & 0x000fffffffffffffull);
}
__global__ void k_corner_keys(const double* __restrict__ C, int64_t n, int k, uint64_t* __restrict__ key,
                              const uint32_t* __restrict__ order) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const uint32_t c = order ? order[j] : static_cast<uint32_t>(j);
  key[j] = static_cast<uint64_t>(__double_as_longlong(C[3 * static_cast<int64_t>(c) + k]));
}
__global__ void k_iota(uint32_t* __restrict__ v, int64_t n) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j < n) v[j] = static_cast<uint32_t>(j);
}
__global__ void k_heads64(const double* __restrict__ C, const uint32_t* __restrict__ idx, int64_t n,
                          uint32_t* __restrict__ head) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const int64_t c = idx[j];
  bool h = j == 0;
  const uint64_t* u = reinterpret_cast<const uint64_t*>(C);
  bool nan = isnan64(u[3 * c]) || isnan64(u[3 * c + 1]) || isnan64(u[3 * c + 2]);
  if (!h) {
    const int64_t d = idx[j - 1];
    nan = nan || isnan64(u[3 * d]) || isnan64(u[3 * d + 1]) || isnan64(u[3 * d + 2]);
    h = u[3 * c] != u[3 * d] || u[3 * c + 1] != u[3 * d + 1] || u[3 * c + 2] != u[3 * d + 2];
  }
  head[j] = (h || nan) ? 1u : 0u;
}
__global__ void k_rep64(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ head,
                        const uint32_t* __restrict__ gid, int64_t n, uint32_t* __restrict__ gfirst) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j < n && head[j]) gfirst[gid[j]] = idx[j];
}
__global__ void k_first64(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ head,
                          const uint32_t* __restrict__ gid, const uint32_t* __restrict__ gfirst, int64_t n,
                          uint32_t* __restrict__ rep, uint32_t* __restrict__ isfirst) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const uint32_t c = idx[j], r = gfirst[gid[j] + head[j] - 1];
  rep[c] = r;
  isfirst[c] = r == c ? 1u : 0u;
}
__global__ void k_emit64(const double* __restrict__ C, const uint32_t* __restrict__ rep,
                         const uint32_t* __restrict__ isfirst, const uint32_t* __restrict__ vpos, int64_t n,
                         double* __restrict__ V, int32_t* __restrict__ tri) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  const uint32_t v = vpos[rep[c]];
  tri[c] = static_cast<int32_t>(v);
  if (isfirst[c])
    for (int k = 0; k < 3; ++k) V[3 * static_cast<int64_t>(v) + k] = C[3 * c + k];
}
__global__ void k_keep_tris(const int32_t* __restrict__ tri, int64_t nf, uint32_t* __restrict__ keep) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const int32_t a = tri[3 * f], b = tri[3 * f + 1], c = tri[3 * f + 2];
  keep[f] = (a != b && b != c && a != c) ? 1u : 0u;
}
__global__ void k_pack_tris(const int32_t* __restrict__ tri, const uint32_t* __restrict__ keep,
                            const uint32_t* __restrict__ pos, int64_t nf, int32_t* __restrict__ out) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f < nf && keep[f])
    for (int k = 0; k < 3; ++k) out[3 * static_cast<int64_t>(pos[f]) + k] = tri[3 * f + k];
}

// StlWelder (mesh_io.cpp:291-301) on 3*nf corners: vertex ids in first-occurrence order, equal
// doubles merged (NaN never equal), then add_polygon's degenerate drop per triangle
void weld_corners64(Ctx& ctx, const std::vector<double>& corners, IngestResult& out) {
  cudaStream_t st = ctx.stream;
  const int64_t n = static_cast<int64_t>(corners.size() / 3), nf = n / 3;
  out = IngestResult();
  if (n == 0) {
    out.V.alloc(1, st);
    out.F.alloc(1, st);
    return;
  }
  DevBuf<double> C(3 * n, st);
  PCU_CUDA(cudaMemcpyAsync(C.get(), corners.data(), 3 * n * 8, cudaMemcpyHostToDevice, st));
  DevBuf<uint64_t> k1(n, st), k2(n, st);
  DevBuf<uint32_t> a(n, st), b(n, st);
  PCU_LAUNCH(ctx, k_iota, grid_for(n, 256), 256, 0, a.get(), n);
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, k1.get(), k2.get(), a.get(), b.get(), static_cast<int>(n), 0, 64, st);
  DevBuf<uint8_t> tmp(need ? need : 1, st);
  // LSD: stable by z, then y, then x -> (x, y, z) order with ties in corner order
  for (int k = 2; k >= 0; --k) {
    PCU_LAUNCH(ctx, k_corner_keys, grid_for(n, 256), 256, 0, C.get(), n, k, k1.get(), a.get());
    PCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), need, k1.get(), k2.get(), a.get(), b.get(),
                                             static_cast<int>(n), 0, 64, st));
    ++ctx.launches;
    std::swap(a, b);
  }
  DevBuf<uint32_t> head(n, st), gid(n, st);
  PCU_LAUNCH(ctx, k_heads64, grid_for(n, 256), 256, 0, C.get(), a.get(), n, head.get());
  exclusive_scan_u32(ctx, head.get(), gid.get(), n);
  const int64_t ng = static_cast<int64_t>(read_scalar(ctx, gid.get() + n - 1)) + read_scalar(ctx, head.get() + n - 1);
  DevBuf<uint32_t> gfirst(ng, st), rep(n, st), isfirst(n, st), vpos(n, st);
  PCU_LAUNCH(ctx, k_rep64, grid_for(n, 256), 256, 0, a.get(), head.get(), gid.get(), n, gfirst.get());
  PCU_LAUNCH(ctx, k_first64, grid_for(n, 256), 256, 0, a.get(), head.get(), gid.get(), gfirst.get(), n, rep.get(),
             isfirst.get());
  exclusive_scan_u32(ctx, isfirst.get(), vpos.get(), n);
  out.nv = ng;
  out.welded = n - ng;
  out.V.alloc(3 * ng, st);
  DevBuf<int32_t> tri(n, st);
  PCU_LAUNCH(ctx, k_emit64, grid_for(n, 256), 256, 0, C.get(), rep.get(), isfirst.get(), vpos.get(), n, out.V.get(),
             tri.get());
  DevBuf<uint32_t> keep(nf, st), pos(nf, st);
  PCU_LAUNCH(ctx, k_keep_tris, grid_for(nf, 256), 256, 0, tri.get(), nf, keep.get());
  exclusive_scan_u32(ctx, keep.get(), pos.get(), nf);
  const int64_t nk = static_cast<int64_t>(read_scalar(ctx, pos.get() + nf - 1)) + read_scalar(ctx, keep.get() + nf - 1);
  out.F.alloc(3 * (nk ? nk : 1), st);
  if (nk) PCU_LAUNCH(ctx, k_pack_tris, grid_for(nf, 256), 256, 0, tri.get(), keep.get(), pos.get(), nf, out.F.get());
  out.nf = nk;
  out.degenerate_dropped = nf - nk;
}

}  // namespace

// ------------------------------------------------------------------------------- OBJ
void load_obj_text(Ctx& ctx, const char* b, int64_t n, IngestResult& out, int64_t* triangulated) {
  HostMesh h;
  for_lines(b, n, [&](std::string_view line, long lineno) {
    Tokens tk{line};
    std::string_view tag;
    if (!tk.next(tag)) return;
    if (tag == "v") {
      double p[3];
      std::string_view t;
      for (int k = 0; k < 3; ++k)
        if (!tk.next(t) || !to_double(t, p[k])) fail("malformed vertex", lineno);
      h.V.insert(h.V.end(), p, p + 3);
    } else if (tag == "f") {
      std::vector<int64_t> poly;
      std::string_view tok;
      while (tk.next(tok)) {
        const std::string_view head = tok.substr(0, tok.find('/'));  // index may carry /vt/vn suffixes
        int idx = 0;
        auto r = std::from_chars(head.data(), head.data() + head.size(), idx);
        if (r.ec != std::errc() || r.ptr != head.data() + head.size())
          fail("malformed face index '" + std::string(tok) + "'", lineno);
        int64_t i = idx < 0 ? h.nv() + idx : static_cast<int64_t>(idx) - 1;  // relative / 1-based
        if (i < 0 || i >= h.nv()) fail("face index out of range", lineno);
        poly.push_back(i);
      }
      if (poly.size() < 3) fail("face with fewer than 3 vertices", lineno);
      h.add_polygon(poly);
    }
  });
  upload(ctx, h, out);
  *triangulated = h.triangulated;
}

// --------------------------------------------------------------------------- ASCII STL
void load_stl_ascii(Ctx& ctx, const char* b, int64_t n, IngestResult& out) {
  std::vector<double> corners;
  Tokens tk{std::string_view(b, static_cast<size_t>(n))};
  std::string_view t;
  long word = 0;
  while (tk.next(t)) {
    ++word;
    if (t != "vertex") continue;
    for (int k = 0; k < 3; ++k) {
      double v;
      if (!tk.next(t) || !to_double(t, v)) fail("malformed vertex at word " + std::to_string(word));
      corners.push_back(v);
    }
  }
  if (corners.size() % 9) fail("dangling vertices at end of ascii stl");
  weld_corners64(ctx, corners, out);
}

// ------------------------------------------------------------------ PLY (host decoder)
// Header + body with the reference's record-by-record semantics (mesh_io.cpp:137-245): ASCII
// bodies, and binary bodies whose face lists vary in length (polygons are fanned).
void load_ply_host(Ctx& ctx, const char* b, int64_t n, IngestResult& out, int64_t* triangulated) {
  struct Prop {
    std::string type, name, count_type;
    bool list = false;
  };
  struct Elem {
    std::string name;
    long count = 0;
    std::vector<Prop> props;
  };
  int64_t p = 0;
  long lineno = 0;
  auto getline = [&](std::string& line) {
    if (p >= n) return false;
    int64_t e = p;
    while (e < n && b[e] != '\n') ++e;
    line.assign(b + p, static_cast<size_t>(e - p));
    p = e + 1;
    return true;
  };
  std::string line;
  if (!getline(line) || line.substr(0, 3) != "ply") fail("missing ply magic", 1);
  ++lineno;
  std::string format;
  std::vector<Elem> els;
  while (getline(line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    Tokens tk{line};
    std::string_view tag, a, c, d;
    if (!tk.next(tag)) continue;
    if (tag == "comment" || tag == "obj_info") continue;
    if (tag == "format") {
      tk.next(a);
      format = std::string(a);
      if (format != "ascii" && format != "binary_little_endian")
        fail("unsupported ply format '" + format + "'", lineno);
    } else if (tag == "element") {
      Elem el;
      tk.next(a);
      el.name = std::string(a);
      if (tk.next(c)) to_int(c, el.count);
      els.push_back(el);
    } else if (tag == "property") {
      if (els.empty()) fail("property before element", lineno);
      Prop pr;
      tk.next(a);
      if (a == "list") {
        pr.list = true;
        tk.next(c);
        tk.next(d);
        pr.count_type = std::string(c);
        pr.type = std::string(d);
        tk.next(a);
        pr.name = std::string(a);
      } else {
        pr.type = std::string(a);
        tk.next(c);
        pr.name = std::string(c);
      }
      els.back().props.push_back(pr);
    } else if (tag == "end_header") {
      break;
    } else {
      fail("unexpected header line '" + std::string(tag) + "'", lineno);
    }
  }
  auto tsize = [](const std::string& t) -> int {
    if (t == "char" || t == "uchar" || t == "int8" || t == "uint8") return 1;
    if (t == "short" || t == "ushort" || t == "int16" || t == "uint16") return 2;
    if (t == "int" || t == "uint" || t == "int32" || t == "uint32" || t == "float" || t == "float32") return 4;
    if (t == "double" || t == "float64") return 8;
    throw Error(PAMOPT_CU_EIO, "unknown ply type: " + t);
  };
  auto bin = [&](const std::string& t, bool& ok) -> double {  // read_binary_scalar (mesh_io.cpp:117-135)
    const int sz = tsize(t);
    if (p + sz > n) {
      ok = false;
      p = n;
      return 0.0;
    }
    unsigned char buf[8];
    std::memcpy(buf, b + p, sz);
    p += sz;
    auto as = [&](auto v) {
      std::memcpy(&v, buf, sizeof(v));
      return static_cast<double>(v);
    };
    if (t == "char" || t == "int8") return as(int8_t{});
    if (t == "uchar" || t == "uint8") return as(uint8_t{});
    if (t == "short" || t == "int16") return as(int16_t{});
    if (t == "ushort" || t == "uint16") return as(uint16_t{});
    if (t == "int" || t == "int32") return as(int32_t{});
    if (t == "uint" || t == "uint32") return as(uint32_t{});
    if (t == "float" || t == "float32") return as(float{});
    return as(double{});
  };
  const bool binary = format == "binary_little_endian";
  HostMesh h;
  for (const Elem& el : els) {
    const bool is_vertex = el.name == "vertex", is_face = el.name == "face";
    int xi = -1, yi = -1, zi = -1;
    for (size_t i = 0; i < el.props.size(); ++i) {
      if (el.props[i].name == "x") xi = static_cast<int>(i);
      if (el.props[i].name == "y") yi = static_cast<int>(i);
      if (el.props[i].name == "z") zi = static_cast<int>(i);
    }
    if (is_vertex && (xi < 0 || yi < 0 || zi < 0)) fail("vertex element lacks x/y/z");
    std::vector<double> sc;
    std::vector<long> list;
    for (long r = 0; r < el.count; ++r) {
      sc.clear();
      list.clear();
      if (binary) {
        bool ok = true;
        for (const Prop& pr : el.props) {
          if (pr.list) {
            const long cnt = static_cast<long>(bin(pr.count_type, ok));
            for (long k = 0; k < cnt && ok; ++k) list.push_back(static_cast<long>(bin(pr.type, ok)));
          } else {
            sc.push_back(bin(pr.type, ok));
          }
        }
        if (!ok) fail("truncated binary body at element '" + el.name + "' row " + std::to_string(r));
      } else {
        if (!getline(line)) fail("truncated ascii body at element '" + el.name + "' row " + std::to_string(r));
        ++lineno;
        Tokens tk{line};
        std::string_view t;
        for (const Prop& pr : el.props) {
          if (pr.list) {
            long cnt = 0;
            if (!tk.next(t) || !to_int(t, cnt)) fail("malformed list count", lineno);
            for (long k = 0; k < cnt; ++k) {
              long v;
              if (!tk.next(t) || !to_int(t, v)) fail("malformed list entry", lineno);
              list.push_back(v);
            }
          } else {
            double v;
            if (!tk.next(t) || !to_double(t, v)) fail("malformed scalar", lineno);
            sc.push_back(v);
          }
        }
      }
      if (is_vertex) {
        h.V.push_back(sc[xi]);
        h.V.push_back(sc[yi]);
        h.V.push_back(sc[zi]);
      } else if (is_face && !list.empty()) {
        std::vector<int64_t> poly;
        for (long v : list) {
          if (v < 0 || v >= h.nv()) fail("face index out of range");
          poly.push_back(v);
        }
        if (poly.size() >= 3) h.add_polygon(poly);
      }
    }
  }
  upload(ctx, h, out);
  *triangulated = h.triangulated;
}

}  // namespace pcu
