// tests/cxx/models_cli.cpp -- the drop-in's analytic models
// (include/wgprof_b200.hpp, perfmodel.hpp:22-222 mirrors) behind the same
// text protocol as oracle/ref_driver.cpp's ref_models, one query per
// NUL-terminated record on stdin, one answer line each on stdout.  Host code
// only: nothing here touches libwgpf.so, so it builds and runs without a GPU.
#include <iostream>
#include <sstream>
#include <string>

#include "wgprof_b200.hpp"

using namespace wgprof;

static std::string dec(const std::string& s) {
  std::string o;
  for (std::size_t i = 0; i < s.size(); ++i) {
    if (s[i] == '%' && i + 2 < s.size()) {
      o.push_back(static_cast<char>(std::stoi(s.substr(i + 1, 2), nullptr, 16)));
      i += 2;
    } else {
      o.push_back(s[i]);
    }
  }
  return o;
}
static std::string enc(const std::string& s) {
  static const char* hx = "0123456789ABCDEF";
  std::string o;
  for (unsigned char c : s) {
    if (c <= ' ' || c == '%' || c >= 0x7F) {
      o += '%';
      o += hx[c >> 4];
      o += hx[c & 15];
    } else {
      o += static_cast<char>(c);
    }
  }
  return o;
}

static std::string answer(const std::string& in) {
  std::ostringstream out;
  try {
    if (in.rfind("table\n", 0) == 0) {
      std::istringstream is(in.substr(6));
      out << "ok";
      for (const auto& x : load_stage_table(is)) out << " " << x.name << " " << x.t_load << " " << x.t_comp;
      return out.str();
    }
    std::istringstream is(in);
    std::string kw;
    SwpInput swp;
    WsInput ws;
    bool is_swp = false, is_ws = false;
    while (is >> kw) {
      if (kw == "swp") {
        is >> swp.n_warp_groups >> swp.n_pipe_stages >> swp.n_loop;
        is_swp = true;
      } else if (kw == "stage") {
        SwpStage st;
        is >> st.name >> st.t_load >> st.t_comp;
        swp.stages.push_back(st);
      } else if (kw == "node") {
        WsNode nd;
        is >> nd.label >> nd.duration;
        nd.label = dec(nd.label);
        ws.nodes.push_back(nd);
        is_ws = true;
      } else if (kw == "edge") {
        std::size_t a, b;
        is >> a >> b;
        ws.edges.emplace_back(a, b);
        is_ws = true;
      } else if (kw == "wsempty") {
        is_ws = true;
      } else if (kw == "roofline") {
        RooflineInput r;
        is >> r.flops >> r.throughput >> r.t_read >> r.bytes >> r.bandwidth;
        const RooflineResult x = roofline(r);
        out << "ok " << x.compute_cycles << " " << x.memory_cycles;
        return out.str();
      } else if (kw == "overhead") {
        OverheadInput o;
        is >> o.t_vanilla >> o.n_record >> o.cycle_record;
        out << "ok " << overhead_model(o);
        return out.str();
      }
    }
    if (is_swp) {
      const SwpResult r = swp_latency(swp);
      out << "ok " << r.delta << " " << r.latency;
    } else if (is_ws) {
      const WsResult r = ws_latency(ws);
      out << "ok " << r.latency;
      for (const auto& l : r.critical_path) out << " " << enc(l);
    } else {
      out << "err none no model";
    }
  } catch (const Error& e) {
    out.str("");
    out << "err " << static_cast<int>(e.kind()) << " " << e.what();
  }
  return out.str();
}

int main() {
  std::string rec;
  while (std::getline(std::cin, rec, '\0')) std::cout << answer(rec) << "\n";
  return 0;
}
