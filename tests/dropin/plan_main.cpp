// Drop-in check (test-side): the reference's planner sources
// (/root/reference/proj/src/optimizer_*.cpp), compiled UNCHANGED against the
// B200 build's headers (include/hetplan/{types,config,memcost,indicator,
// latcost}.hpp) and linked against libhetplan_b200.so, must produce the same
// plan as the reference build. latcost's predictions come from the build's
// Eigen-free latcost.cpp (the reference's needs Eigen, absent here).
#include <fstream>
#include <iostream>
#include <sstream>

#include <json.hpp>

#include "hetplan/config.hpp"
#include "hetplan/indicator/indicator.hpp"
#include "hetplan/optimizer/planner.hpp"

static std::string slurp(const char* p) {
    std::ifstream f(p);
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    auto rs = hetplan::parse_config(slurp(argv[1]));
    auto omega = hetplan::indicator::parse_indicator_table(slurp(argv[2]));
    hetplan::latcost::latency_model lat;
    auto lj = nlohmann::json::parse(slurp(argv[3]));
    for (auto& [dev, per_bit] : lj.items())
        for (auto& [bit, ph] : per_bit.items()) {
            lat.coeffs[{dev, std::stoi(bit), hetplan::latcost::phase::prefill}] =
                ph.at("prefill").get<std::vector<double>>();
            lat.coeffs[{dev, std::stoi(bit), hetplan::latcost::phase::decode}] =
                ph.at("decode").get<std::vector<double>>();
        }
    hetplan::optimizer::plan_options opt;
    opt.theta = 0.001;
    opt.time_limit_s = 5.0;
    auto res = hetplan::optimizer::best_plan(rs.model, rs.cluster, rs.load, rs.bits, lat, omega, opt);
    if (!res.feasible) return 3;
    std::cout << "eta " << res.best.eta << " xi " << res.best.xi << " optimal " << res.optimal << "\nbits";
    for (int b : res.best.layer_bits) std::cout << ' ' << b;
    std::cout << "\nstages";
    for (auto& s : res.best.stages) std::cout << ' ' << s.begin << '-' << s.end;
    std::cout << "\n";
    return 0;
}
