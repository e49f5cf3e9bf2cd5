// Command-line access to the VERBATIM reference IO (proj/src/io.cpp), built
// into oracle/_ref/io_ref by oracle/Makefile. TEST INFRASTRUCTURE ONLY: the
// IO parity tests (tests/test_io_cpu.py) drive it to check the Python host
// mirror (paper_2005_10123_b200/io.py) against the reference's readEvents,
// writeEvents, deduplicate, writeChain, readChain and loadRunConfig.
//
// Every command prints one JSON object on stdout: {"ok": true, ...} or
// {"ok": false, "type": "runtime_error"|"invalid_argument", "what": "..."}.
// Doubles travel as C99 hex strings (lossless).
//
//   io_ref read PATH DELIM XCOL YCOL TCOL DIST TIME REF [WINDOW_END]
//   io_ref write EVENTS_JSON OUT_PATH            (optional "parent" array)
//   io_ref dedup EVENTS_JSON RADIUS_KM WINDOW_DAYS
//   io_ref chain N ITERS SEED OUT_PATH           (runChain on a small cloud, writeChain)
//   io_ref readchain PATH
//   io_ref config PATH
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>

#include <json.hpp>

#include "sthawkes/io.hpp"
#include "sthawkes/rng.hpp"
#include "sthawkes/sampler.hpp"
#include "sthawkes/simulate.hpp"

using namespace hawkes;
using nlohmann::json;

namespace {

std::string hx(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%a", v);
  return buf;
}

double unhx(const json& j) { return std::strtod(j.get<std::string>().c_str(), nullptr); }

json eventsJson(const EventSet& e) {
  json x = json::array(), y = json::array(), t = json::array();
  for (Index i = 0; i < e.size(); ++i) {
    x.push_back(hx(e.xs()[i]));
    y.push_back(hx(e.ys()[i]));
    t.push_back(hx(e.ts()[i]));
  }
  return json{{"ok", true}, {"x", x}, {"y", y}, {"t", t}, {"windowEnd", hx(e.windowEnd())},
              {"timeOrigin", hx(e.timeOrigin())}};
}

EventSet eventsFrom(const json& j) {
  const size_t n = j.at("x").size();
  Eigen::ArrayXd x(static_cast<Index>(n)), y(static_cast<Index>(n)), t(static_cast<Index>(n));
  for (size_t i = 0; i < n; ++i) {
    x[static_cast<Index>(i)] = unhx(j["x"][i]);
    y[static_cast<Index>(i)] = unhx(j["y"][i]);
    t[static_cast<Index>(i)] = unhx(j["t"][i]);
  }
  return EventSet(std::move(x), std::move(y), std::move(t), unhx(j.at("windowEnd")),
                  unhx(j.at("timeOrigin")));
}

json readJson(const std::string& path) {
  std::ifstream in(path);
  json j;
  in >> j;
  return j;
}

json chainJson(const Chain& c) {
  json draws = json::array(), lp = json::array(), ad = json::array();
  for (Index i = 0; i < c.draws.rows(); ++i) {
    json row = json::array();
    for (int d = 0; d < kFreeParams; ++d) row.push_back(hx(c.draws(i, d)));
    draws.push_back(row);
    lp.push_back(hx(c.logPost[i]));
  }
  for (const auto& a : c.adaptations) {
    ad.push_back(json{{"step", a.step}, {"coord", a.coord}, {"v", hx(a.vAfter)},
                      {"b", hx(a.bAfter)}});
  }
  json it = json::array(), ps = json::array();
  for (int d = 0; d < kFreeParams; ++d) {
    it.push_back(hx(c.config.initialTheta[d]));
    ps.push_back(hx(c.config.initialProposalSd[d]));
  }
  json pri = json::array();
  for (const auto& p : c.priors.coord) pri.push_back(json::array({hx(p.mean), hx(p.sd)}));
  return json{{"ok", true},
              {"chainIndex", c.chainIndex},
              {"chainSeed", c.chainSeed},
              {"eventCount", c.eventCount},
              {"iterations", c.config.iterations},
              {"burnIn", c.config.burnIn},
              {"seed", c.config.seed},
              {"targetAcceptance", hx(c.config.targetAcceptance)},
              {"initialTheta", it},
              {"initialProposalSd", ps},
              {"initialAdaptBound", hx(c.config.initialAdaptBound)},
              {"adapt", c.config.adapt},
              {"tauX", hx(c.config.tauX)},
              {"tauT", hx(c.config.tauT)},
              {"backend", json::array({static_cast<int>(c.config.backend.kind),
                                       c.config.backend.threadCount,
                                       c.config.backend.laneWidth})},
              {"chainCount", c.config.chainCount},
              {"priors", pri},
              {"draws", draws},
              {"logPost", lp},
              {"scannedCoord", c.scannedCoord},
              {"accepted", c.accepted},
              {"adaptations", ad}};
}

}  // namespace

int main(int argc, char** argv) {
  json out;
  try {
    if (argc < 2) throw std::invalid_argument("usage: io_ref COMMAND ...");
    const std::string cmd = argv[1];
    if (cmd == "read" && argc >= 10) {
      EventFileSpec spec;
      spec.delimiter = argv[3][0];
      spec.xColumn = argv[4];
      spec.yColumn = argv[5];
      spec.tColumn = argv[6];
      spec.distanceUnit = parseDistanceUnit(argv[7]);
      spec.timeUnit = parseTimeUnit(argv[8]);
      spec.timeReference = std::string(argv[9]) == "epoch" ? TimeReference::Epoch
                                                           : TimeReference::WindowRelative;
      if (argc >= 11) spec.windowEndDays = std::strtod(argv[10], nullptr);
      out = eventsJson(readEvents(argv[2], spec));
    } else if (cmd == "write" && argc >= 4) {
      const json j = readJson(argv[2]);
      const EventSet e = eventsFrom(j);
      if (j.contains("parent")) {
        Eigen::VectorXi par(static_cast<Index>(j["parent"].size()));
        for (size_t i = 0; i < j["parent"].size(); ++i) {
          par[static_cast<Index>(i)] = j["parent"][i].get<int>();
        }
        writeEvents(e, argv[3], &par);
      } else {
        writeEvents(e, argv[3]);
      }
      out = json{{"ok", true}};
    } else if (cmd == "dedup" && argc >= 5) {
      const EventSet e = eventsFrom(readJson(argv[2]));
      out = eventsJson(deduplicate(e, std::strtod(argv[3], nullptr), std::strtod(argv[4], nullptr)));
    } else if (cmd == "chain" && argc >= 6) {
      const Index n = std::atol(argv[2]);
      Rng rng(11);
      const EventSet e = generateBenchmarkCloud(n, SimWindow{0, 4, 0, 4, 60}, rng);
      SamplerConfig cfg;
      cfg.iterations = std::atol(argv[3]);
      cfg.burnIn = cfg.iterations / 10;
      cfg.seed = std::strtoull(argv[4], nullptr, 10);
      const Chain c = runChain(e, PriorSpec{}, cfg);
      writeChain(c, argv[5]);
      out = chainJson(c);
    } else if (cmd == "readchain" && argc >= 3) {
      out = chainJson(readChain(argv[2]));
    } else if (cmd == "config" && argc >= 3) {
      const RunConfig rc = loadRunConfig(argv[2]);
      json it = json::array(), ps = json::array(), pri = json::array();
      for (int d = 0; d < kFreeParams; ++d) {
        it.push_back(hx(rc.sampler.initialTheta[d]));
        ps.push_back(hx(rc.sampler.initialProposalSd[d]));
      }
      for (const auto& p : rc.priors.coord) pri.push_back(json::array({hx(p.mean), hx(p.sd)}));
      out = json{{"ok", true},
                 {"dataPath", rc.dataPath},
                 {"delimiter", std::string(1, rc.fileSpec.delimiter)},
                 {"xColumn", rc.fileSpec.xColumn},
                 {"yColumn", rc.fileSpec.yColumn},
                 {"tColumn", rc.fileSpec.tColumn},
                 {"distanceUnit", static_cast<int>(rc.fileSpec.distanceUnit)},
                 {"timeUnit", static_cast<int>(rc.fileSpec.timeUnit)},
                 {"timeReference", static_cast<int>(rc.fileSpec.timeReference)},
                 {"windowEndDays", rc.fileSpec.windowEndDays ? hx(*rc.fileSpec.windowEndDays)
                                                             : std::string("none")},
                 {"dedupRadiusKm", hx(rc.dedup.radiusKm)},
                 {"dedupWindowDays", hx(rc.dedup.windowDays)},
                 {"iterations", rc.sampler.iterations},
                 {"burnIn", rc.sampler.burnIn},
                 {"seed", rc.sampler.seed},
                 {"chainCount", rc.sampler.chainCount},
                 {"targetAcceptance", hx(rc.sampler.targetAcceptance)},
                 {"adapt", rc.sampler.adapt},
                 {"initialTheta", it},
                 {"initialProposalSd", ps},
                 {"tauX", hx(rc.sampler.tauX)},
                 {"tauT", hx(rc.sampler.tauT)},
                 {"backend", json::array({static_cast<int>(rc.sampler.backend.kind),
                                          rc.sampler.backend.threadCount,
                                          rc.sampler.backend.laneWidth})},
                 {"priors", pri},
                 {"outputPrefix", rc.outputPrefix}};
    } else {
      throw std::invalid_argument("io_ref: bad command line");
    }
  } catch (const std::invalid_argument& e) {
    out = json{{"ok", false}, {"type", "invalid_argument"}, {"what", e.what()}};
  } catch (const std::exception& e) {
    out = json{{"ok", false}, {"type", "runtime_error"}, {"what", e.what()}};
  }
  std::cout << out.dump() << "\n";
  return 0;
}
