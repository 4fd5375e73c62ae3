// b200_report.cpp -- drives the REFERENCE's own analysis pipeline over timing
// logs measured on a B200.  TEST / EVIDENCE
// INFRASTRUCTURE: compiled by oracle/Makefile together with the reference's
// src/timing_log.cpp, analyzer.cpp, exec_model.cpp, report.cpp and svg.cpp,
// straight from /root/reference (never copied), into oracle/_ref/.
//
// It replaces only the reference CLI's `analyze` front end
// (proj/src/cli.cpp:220-250), which needs CLI11 and nlohmann/json -- both
// absent from the reference tree.  The device spec is read from a flat JSON
// object with the reference's DeviceSpec field names
// (proj/src/device_spec.cpp:50-78) by the small parser below; everything
// after that is the reference's code: parse_timing_csv
// (src/timing_log.cpp:33-97), build_report (src/report.cpp:36-94) and the
// deterministic writers.
//
// usage: ks_b200_report <timing.csv> <device_spec.json> B H L K <out_dir>
// writes <out_dir>/{report.txt,speedups.csv,bandwidth.csv,roofline.csv,roofline.svg}
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <regex>
#include <sstream>
#include <string>

#include "kernelscope/report.hpp"
#include "kernelscope/svg.hpp"
#include "kernelscope/timing_log.hpp"

namespace {

std::string slurp(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::ostringstream s;
    s << in.rdbuf();
    return s.str();
}

// Flat {"key": number | "string", ...} objects only (the DeviceSpec schema).
std::string field(const std::string& j, const std::string& key) {
    const std::regex re("\"" + key + "\"\\s*:\\s*(\"([^\"]*)\"|[-+0-9.eE]+)");
    std::smatch m;
    if (!std::regex_search(j, m, re)) throw std::runtime_error("device spec: missing field '" + key + "'");
    return m[2].matched ? m[2].str() : m[1].str();
}

kernelscope::DeviceSpec parse_spec(const std::string& j) {
    kernelscope::DeviceSpec d;
    d.name = field(j, "name");
    d.sm_count = std::stoll(field(j, "sm_count"));
    d.warp_size = std::stoll(field(j, "warp_size"));
    d.max_threads_per_block = std::stoll(field(j, "max_threads_per_block"));
    d.max_threads_per_sm = std::stoll(field(j, "max_threads_per_sm"));
    d.smem_per_block = std::stoll(field(j, "smem_per_block"));
    d.smem_per_sm = std::stoll(field(j, "smem_per_sm"));
    d.registers_per_sm = std::stoll(field(j, "registers_per_sm"));
    d.l2_bytes = std::stoll(field(j, "l2_bytes"));
    d.mem_bytes = std::stoll(field(j, "mem_bytes"));
    d.peak_bw = std::stod(field(j, "peak_bw"));
    d.peak_fp32 = std::stod(field(j, "peak_fp32"));
    return d;
}

void write(const std::string& path, const std::string& text) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write " + path);
    out << text;
}

}  // namespace

int main(int argc, char** argv) {
    using namespace kernelscope;
    if (argc != 8) {
        std::cerr << "usage: ks_b200_report <timing.csv> <device_spec.json> B H L K <out_dir>\n";
        return 2;
    }
    try {
        const cli::TimingLog log = cli::load_timing_csv(argv[1]);
        const DeviceSpec dev = parse_spec(slurp(argv[2]));
        const ConvShape shape(std::atoll(argv[3]), std::atoll(argv[4]), std::atoll(argv[5]), std::atoll(argv[6]));
        cli::Provenance prov;
        prov.timing_csv = argv[1];
        prov.device_spec = argv[2];
        prov.shape = shape;
        const cli::ReportBundle b = cli::build_report(log, dev, shape, prov);
        const std::string dir = argv[7];
        std::ostringstream sp, bw, rl, txt, svg;
        cli::write_speedups_csv(sp, b);
        cli::write_bandwidth_csv(bw, b);
        cli::write_roofline_csv(rl, b);
        cli::write_report_txt(txt, b, dev);
        cli::write_roofline_svg(svg, b.roofline, dev);
        write(dir + "/speedups.csv", sp.str());
        write(dir + "/bandwidth.csv", bw.str());
        write(dir + "/roofline.csv", rl.str());
        write(dir + "/report.txt", txt.str());
        write(dir + "/roofline.svg", svg.str());
        std::cout << txt.str();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
