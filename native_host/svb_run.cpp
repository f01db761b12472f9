// Native host for the B200 executor: runs a compiled
// device program without Python.
//
//   svb_run <program.svbp> <plan.json> <out.bin>
//
// The program file (paper_2509_14098_b200/program_file.py) holds the sweep
// descriptors, the program blob and the generated CUDA source of every sweep
// kernel; the plan is the reference's JSON wire format
// (svpart/plan.py:171-201).  The task loop follows svpart/executor.py:179-307:
// the same dependency and protocol checks (exit code 2 = PlanInvalid), sweeps
// launched through include/svb200.h (NVRTC compile + load + launch), the norm
// of every ApplyFused leaf checked at the end (exit code 3 =
// NonUnitaryDrift, |norm - 1| > 1e-8).  One device holds every rank, so
// remaps are relabels the program already folded into its layouts.  The
// final rank blocks (2^g x 2^L complex128, reference layout) are written to
// out.bin.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "svb200.h"

namespace {

[[noreturn]] void die(int code, const std::string& msg) {
  std::fprintf(stderr, "svb_run: %s\n", msg.c_str());
  std::exit(code);
}

void check(int rc, const char* what) {
  if (rc != SVB_OK) die(1, std::string(what) + ": " + svb_last_error());
}

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) die(1, std::string(what) + ": " + cudaGetErrorString(e));
}

std::string slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) die(1, std::string("cannot read ") + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// ---- minimal JSON (the plan wire format) ---------------------------------
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json& operator[](const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return kv.second;
    static Json none;
    return none;
  }
  std::string dump() const {  // canonical re-serialisation (payload equality)
    std::ostringstream o;
    switch (kind) {
      case Null: o << "null"; break;
      case Bool: o << (b ? "true" : "false"); break;
      case Num: o << num; break;
      case Str: o << '"' << str << '"'; break;
      case Arr:
        o << '[';
        for (size_t i = 0; i < arr.size(); ++i) o << (i ? "," : "") << arr[i].dump();
        o << ']';
        break;
      case Obj:
        o << '{';
        for (size_t i = 0; i < obj.size(); ++i) o << (i ? "," : "") << '"' << obj[i].first << "\":" << obj[i].second.dump();
        o << '}';
        break;
    }
    return o.str();
  }
};

struct Parser {
  const std::string& s;
  size_t i = 0;
  void ws() {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
  }
  Json value() {
    ws();
    if (i >= s.size()) die(1, "plan JSON: unexpected end");
    Json v;
    const char c = s[i];
    if (c == '{') {
      v.kind = Json::Obj;
      ++i;
      ws();
      if (s[i] == '}') {
        ++i;
        return v;
      }
      while (true) {
        ws();
        std::string k = string();
        ws();
        if (s[i++] != ':') die(1, "plan JSON: expected ':'");
        v.obj.emplace_back(k, value());
        ws();
        if (s[i] == ',') {
          ++i;
          continue;
        }
        if (s[i++] != '}') die(1, "plan JSON: expected '}'");
        return v;
      }
    }
    if (c == '[') {
      v.kind = Json::Arr;
      ++i;
      ws();
      if (s[i] == ']') {
        ++i;
        return v;
      }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (s[i] == ',') {
          ++i;
          continue;
        }
        if (s[i++] != ']') die(1, "plan JSON: expected ']'");
        return v;
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      v.str = string();
      return v;
    }
    if (!s.compare(i, 4, "true")) {
      i += 4;
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (!s.compare(i, 5, "false")) {
      i += 5;
      v.kind = Json::Bool;
      return v;
    }
    if (!s.compare(i, 4, "null")) {
      i += 4;
      return v;
    }
    char* end = nullptr;
    v.kind = Json::Num;
    v.num = std::strtod(s.c_str() + i, &end);
    if (end == s.c_str() + i) die(1, "plan JSON: bad value");
    i = end - s.c_str();
    return v;
  }
  std::string string() {
    if (s[i++] != '"') die(1, "plan JSON: expected string");
    std::string out;
    while (s[i] != '"') {
      if (s[i] == '\\') ++i;
      out += s[i++];
    }
    ++i;
    return out;
  }
};

// ---- program file ---------------------------------------------------------
struct Program {
  int d, g, L, D, rows, n_fused, sparse, nsteps, ndescs, nkernels, unit;
  std::string blob;
  std::vector<svb_sweep_desc> descs;
  struct Step {
    int kind, task_id, first, count, nremote;
  };
  std::vector<Step> steps;
  std::vector<int> alias;
  std::vector<std::pair<std::string, std::string>> kernels;  // name, source
  std::vector<std::string> opts;
};

Program load_program(const char* path) {
  const std::string raw = slurp(path);
  if (raw.size() < 8 || raw.compare(0, 4, "SVBP")) die(1, "not a program file");
  uint32_t ver;
  std::memcpy(&ver, raw.data() + 4, 4);
  if (ver != 1) die(1, "program file version");
  std::map<std::string, std::string> sec;
  size_t off = 8;
  while (off + 12 <= raw.size()) {
    const std::string tag = raw.substr(off, 4);
    uint64_t n;
    std::memcpy(&n, raw.data() + off + 4, 8);
    sec[tag] = raw.substr(off + 12, n);
    off += 12 + n;
  }
  Program p;
  const std::string& h = sec["HEAD"];
  if (h.size() != 11 * 4) die(1, "HEAD section");
  int hv[11];
  std::memcpy(hv, h.data(), sizeof(hv));
  p.d = hv[0], p.g = hv[1], p.L = hv[2], p.D = hv[3], p.rows = hv[4], p.n_fused = hv[5], p.sparse = hv[6];
  p.nsteps = hv[7], p.ndescs = hv[8], p.nkernels = hv[9], p.unit = hv[10];
  p.blob = sec["BLOB"];
  size_t a = 0, b = 0, c = 0;
  svb_abi_sizes(&a, &b, &c);
  if (sec["DESC"].size() != c * (size_t)p.ndescs) die(1, "DESC section size (ABI mismatch?)");
  p.descs.resize(p.ndescs);
  std::memcpy(p.descs.data(), sec["DESC"].data(), sec["DESC"].size());
  p.steps.resize(p.nsteps);
  std::memcpy(p.steps.data(), sec["STEP"].data(), sizeof(Program::Step) * p.nsteps);
  p.alias.resize(p.n_fused);
  std::memcpy(p.alias.data(), sec["ALIA"].data(), 4 * p.n_fused);
  const std::string& k = sec["KERN"];
  size_t q = 0;
  for (int i = 0; i < p.nkernels; ++i) {
    uint32_t n1, n2;
    std::memcpy(&n1, k.data() + q, 4);
    std::string name = k.substr(q + 4, n1);
    q += 4 + n1;
    std::memcpy(&n2, k.data() + q, 4);
    std::string src = k.substr(q + 4, n2);
    q += 4 + n2;
    p.kernels.emplace_back(name, src);
  }
  const std::string& o = sec["OPTS"];
  uint32_t no;
  std::memcpy(&no, o.data(), 4);
  size_t r = 4;
  for (uint32_t i = 0; i < no; ++i) {
    uint32_t n;
    std::memcpy(&n, o.data() + r, 4);
    p.opts.push_back(o.substr(r + 4, n));
    r += 4 + n;
  }
  return p;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 4) die(1, "usage: svb_run <program.svbp> <plan.json> <out.bin>");
  const Program prog = load_program(argv[1]);
  const std::string ptxt = slurp(argv[2]);
  Parser pp{ptxt};
  const Json plan = pp.value();
  if ((int)plan["d"].num != prog.d || (int)plan["g"].num != prog.g) die(1, "plan and program disagree on d/g");
  const int64_t nranks = int64_t(1) << prog.g;
  const int64_t n_amp = int64_t(1) << prog.D;

  // kernels: NVRTC through the C ABI
  std::vector<const char*> opts;
  for (auto& o : prog.opts) opts.push_back(o.c_str());
  std::vector<void*> kern(prog.nkernels);
  std::vector<char> log(1 << 16);
  for (int i = 0; i < prog.nkernels; ++i) {
    void* image = nullptr;
    size_t size = 0;
    int rc = svb_jit_compile(prog.kernels[i].second.c_str(), prog.kernels[i].first.c_str(), (int)opts.size(),
                             opts.data(), &image, &size, log.data(), log.size());
    if (rc != SVB_OK) die(1, "NVRTC: " + std::string(log.data()));
    check(svb_jit_load(image, prog.kernels[i].first.c_str(), &kern[i]), "svb_jit_load");
    svb_jit_free(image);
  }
  std::map<int, const Program::Step*> by_task;
  const Program::Step* materialize = nullptr;
  for (auto& st : prog.steps) {
    if (st.kind == 2)
      materialize = &st;
    else if (st.task_id >= 0)
      by_task[st.task_id] = &st;
  }

  cudaStream_t stream;
  cuda(cudaStreamCreate(&stream), "stream");
  void* blob = nullptr;
  cuda(cudaMalloc(&blob, prog.blob.size()), "blob");
  cuda(cudaMemcpy(blob, prog.blob.data(), prog.blob.size(), cudaMemcpyHostToDevice), "blob copy");
  svb_c128* state = nullptr;
  double* norms = nullptr;
  cuda(cudaMalloc(&norms, sizeof(double) * (prog.n_fused + 1)), "norms");
  cuda(cudaMemset(norms, 0, sizeof(double) * (prog.n_fused + 1)), "norms");

  auto launch = [&](int first, int count, double* nptr) {
    for (int i = first; i < first + count; ++i)
      check(svb_jit_launch_sweep(kern[i], state, blob, &prog.descs[i], nptr, 0, stream), "svb_jit_launch_sweep");
  };

  std::set<int> done;
  bool allocated = false, pending = false, sent = false;
  std::string pack_swaps;
  int slot = 0;
  for (const Json& t : plan["tasks"].arr) {
    const int id = (int)t["id"].num;
    const std::string kind = t["kind"].str;
    for (const Json& dep : t["deps"].arr)
      if (!done.count((int)dep.num)) die(2, "PlanInvalid: task " + std::to_string(id) + " runs before its dependencies");
    if (kind == "Alloc") {
      if (allocated) die(2, "PlanInvalid: double Alloc");
      if ((int64_t)t["payload"]["num_ranks"].num != nranks ||
          (int64_t)t["payload"]["block_len"].num != (int64_t(1) << prog.L))
        die(2, "PlanInvalid: Alloc payload disagrees with plan shape");
      cuda(cudaMalloc(&state, 16 * n_amp), "state");
      if (!prog.sparse) {  // |0...0>: index 0 in every layout
        cuda(cudaMemsetAsync(state, 0, 16 * n_amp, stream), "memset");
        const double one[2] = {1.0, 0.0};
        cuda(cudaMemcpyAsync(state, one, 16, cudaMemcpyHostToDevice, stream), "unit");
      }
      allocated = true;
    } else if (kind == "ApplyFused") {
      if (!allocated) die(2, "PlanInvalid: compute before Alloc");
      auto it = by_task.find(id);
      if (it == by_task.end()) die(1, "program has no step for task " + std::to_string(id));
      const Program::Step& st = *it->second;
      if (st.count) {
        launch(st.first, st.count, norms);
      } else if (prog.alias[slot] < 0) {  // no sweep yet: the norm of |0...0>
        const double one = 1.0;
        cuda(cudaMemcpyAsync(norms + slot, &one, 8, cudaMemcpyHostToDevice, stream), "norm");
      }
      ++slot;
    } else if (kind == "Pack") {
      if (!allocated) die(2, "PlanInvalid: Pack before Alloc");
      if (pending) die(2, "PlanInvalid: Pack while a previous Pack is pending");
      pending = true;
      sent = false;
      pack_swaps = t["payload"]["swaps"].dump();
    } else if (kind == "Exchange") {
      if (!pending || t["payload"]["swaps"].dump() != pack_swaps) die(2, "PlanInvalid: Exchange without matching Pack");
      auto it = by_task.find(id);
      if (it != by_task.end() && it->second->nremote) die(1, "remote remap: this host drives one device");
      sent = true;  // ranks on one device: the program relabelled the bits
    } else if (kind == "Unpack") {
      if (!pending || !sent) die(2, "PlanInvalid: Unpack without a completed Exchange");
      pending = false;
    } else if (kind == "Free") {
      if (pending) die(2, "PlanInvalid: Free with undelivered messages");
    } else {
      die(2, "PlanInvalid: unknown task kind " + kind);
    }
    done.insert(id);
  }
  if (!allocated) die(2, "PlanInvalid: plan never allocated state");
  if (materialize) launch(materialize->first, materialize->count, nullptr);
  cuda(cudaStreamSynchronize(stream), "run");
  std::vector<double> nv(prog.n_fused + 1);
  cuda(cudaMemcpy(nv.data(), norms, sizeof(double) * nv.size(), cudaMemcpyDeviceToHost), "norms");
  for (int s = 0; s < prog.n_fused; ++s) {
    const double v = nv[prog.alias[s] >= 0 ? prog.alias[s] : s];
    if (std::fabs(v - 1.0) > 1e-8) {
      char msg[128];
      std::snprintf(msg, sizeof(msg), "NonUnitaryDrift: norm drifted to %.17g", v);
      die(3, msg);
    }
  }
  std::vector<svb_c128> host(nranks << prog.L);
  cuda(cudaMemcpy(host.data(), state, 16 * host.size(), cudaMemcpyDeviceToHost), "download");
  std::ofstream out(argv[3], std::ios::binary);
  out.write(reinterpret_cast<const char*>(host.data()), 16 * host.size());
  std::printf("svb_run: %s d=%d g=%d sweeps=%d kernels=%d ok\n", argv[1], prog.d, prog.g, prog.ndescs,
              prog.nkernels);
  return 0;
}
