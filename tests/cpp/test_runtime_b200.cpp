// C++ runtime tests against include/manta_b200.hpp, written like the reference's own
// proj/tests/unit/test_runtime.cpp (same scenarios, same expected values). Needs a GPU.
#include <cstdio>
#include <cstring>
#include <dlfcn.h>
#include <limits>

#include "../../include/manta_b200.hpp"

using namespace manta_b200;

static int failures = 0;
#define CHECK(cond)                                                                        \
	do {                                                                                   \
		if(!(cond)) {                                                                      \
			std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
			++failures;                                                                    \
		}                                                                                  \
	} while(0)

// paper-style iterated stencil through the full driver + runtime (test_runtime.cpp:45-65)
static std::vector<float> run_stencil(int workers, int devices, int iterations, int64_t n) {
	driver drv({workers, devices, false, false, true, 1});
	const auto devs = drv.devices();
	const rect dom({0}, {n});
	auto in = drv.create_array(dom, dtype::f32, stencil_dist(dom, {n / 8}, {1}, devs), fill_spec::one());
	auto out = drv.create_array(dom, dtype::f32, stencil_dist(dom, {n / 8}, {1}, devs), fill_spec::zero());
	drv.flush();
	const auto work = block_work_dist(dom, {16}, {n / 8}, devs);
	for(int it = 0; it < iterations; ++it) {
		drv.launch("stencil1d", dom, {16}, work, {launch_arg::scalar(n), launch_arg::array(out), launch_arg::array(in)},
		    "global i => read input[i-1:i+1], write output[i]");
		drv.flush();
		std::swap(in, out);
	}
	drv.synchronize();
	return drv.read<float>(in, static_cast<size_t>(n));
}

// the same stencil with device, pinned-host and disk tiers all in play (memory_config,
// memory.hpp:43-55): spill traffic must reach the disk tier and the result stay bit-exact
static std::vector<float> run_stencil_tiered(int iterations, int64_t n, std::string* report) {
	driver_config cfg{1, 1, false, false, true, 1};
	const uint64_t chunk = static_cast<uint64_t>(n / 8 + 2) * sizeof(float);
	cfg.memory.device_capacity = 4 * chunk;
	cfg.memory.host_capacity = 4 * chunk;
	cfg.memory.disk_capacity = 64 * chunk;
	driver drv(cfg);
	const auto devs = drv.devices();
	const rect dom({0}, {n});
	auto in = drv.create_array(dom, dtype::f32, stencil_dist(dom, {n / 8}, {1}, devs), fill_spec::one());
	auto out = drv.create_array(dom, dtype::f32, stencil_dist(dom, {n / 8}, {1}, devs), fill_spec::zero());
	drv.flush();
	const auto work = block_work_dist(dom, {16}, {n / 8}, devs);
	for(int it = 0; it < iterations; ++it) {
		drv.launch("stencil1d", dom, {16}, work, {launch_arg::scalar(n), launch_arg::array(out), launch_arg::array(in)},
		    "global i => read input[i-1:i+1], write output[i]");
		drv.flush();
		std::swap(in, out);
	}
	drv.synchronize();
	*report = drv.report_json();
	return drv.read<float>(in, static_cast<size_t>(n));
}

int main() {
	// device + host + disk tiers (B200 memory_config): bit-exact against the unconstrained run
	{
		std::string report;
		const auto tiered = run_stencil_tiered(6, 1 << 20, &report);
		const auto plain = run_stencil(1, 1, 6, 1 << 20);
		CHECK(std::memcmp(tiered.data(), plain.data(), plain.size() * sizeof(float)) == 0);
		CHECK(report.find("\"bytes_host_to_disk\": 0,") == std::string::npos);
		CHECK(report.find("\"bytes_host_to_disk\"") != std::string::npos);
	}
	// distributed stencil equals the single-device serial run (test_runtime.cpp:67-72), bit-exact
	{
		const auto serial = run_stencil(1, 1, 4, 4096);
		const auto distributed = run_stencil(2, 2, 4, 4096);
		CHECK(std::memcmp(serial.data(), distributed.data(), serial.size() * sizeof(float)) == 0);
		CHECK(serial[0] < 1.0f && serial[100] == 1.0f);
	}
	// matmul of all-ones is k everywhere (test_runtime.cpp:95-119)
	{
		driver drv({2, 2, false, false, true, 1});
		const auto devs = drv.devices();
		const rect dom({0, 0}, {32, 32});
		const auto a = drv.create_array(dom, dtype::f32, row_dist(dom, 8, devs), fill_spec::one());
		const auto b = drv.create_array(dom, dtype::f32, row_dist(dom, 8, devs), fill_spec::one());
		const auto c = drv.create_array(dom, dtype::f32, row_dist(dom, 8, devs), fill_spec::zero());
		drv.launch("matmul", dom, {8, 8}, block_work_dist(dom, {8, 8}, {8, 32}, devs),
		    {launch_arg::scalar(int64_t{32}), launch_arg::scalar(int64_t{32}), launch_arg::scalar(int64_t{32}), launch_arg::array(c), launch_arg::array(a),
		        launch_arg::array(b)},
		    "global [i, j] => write C[i,j], read A[i,:], read B[:,j]");
		const auto v = drv.read<float>(c, 32 * 32);
		bool all = true;
		for(float x : v) all = all && x == 32.0f;
		CHECK(all);
	}
	// column-sum reduction of an all-ones matrix (test_runtime.cpp:121-157)
	{
		driver drv({2, 2, false, false, true, 1});
		const auto devs = drv.devices();
		const rect mat({0, 0}, {8, 8});
		const rect vec({0}, {8});
		const auto a = drv.create_array(mat, dtype::i64, row_dist(mat, 4, devs), fill_spec::one());
		const auto sum = drv.create_array(vec, dtype::i64, single_dist(vec, devs[0]), fill_spec::zero());
		drv.launch("row_reduce_i64", mat, {2, 2}, block_work_dist(mat, {2, 2}, {8, 4}, devs),
		    {launch_arg::scalar(int64_t{8}), launch_arg::scalar(int64_t{8}), launch_arg::array(a), launch_arg::array(sum)},
		    "global [i, j] => read A[i,j], reduce(+) sum[i]");
		const auto v = drv.read<int64_t>(sum, 8);
		for(int i = 0; i < 8; ++i) CHECK(v[static_cast<size_t>(i)] == 8);
	}
	// reduce(min) leaves untouched cells at type-max (test_runtime.cpp:159-194)
	{
		driver drv({1, 1, false, false, true, 1});
		const auto devs = drv.devices();
		const rect vec({0}, {8});
		const auto src = drv.create_array(vec, dtype::i64, single_dist(vec, devs[0]), fill_spec::one());
		const auto dst = drv.create_array(vec, dtype::i64, single_dist(vec, devs[0]), fill_spec::zero());
		drv.launch("partial_min", vec, {2}, block_work_dist(vec, {2}, {8}, devs), {launch_arg::scalar(int64_t{8}), launch_arg::array(src), launch_arg::array(dst)},
		    "global i => read src[i], reduce(min) dst[:]");
		const auto v = drv.read<int64_t>(dst, 8);
		for(int i = 0; i < 4; ++i) CHECK(v[static_cast<size_t>(i)] == 1 + i);
		for(int i = 4; i < 8; ++i) CHECK(v[static_cast<size_t>(i)] == std::numeric_limits<int64_t>::max());
	}
	// error kinds (errors.hpp): unknown kernel -> plan_error, nonlinear -> parse_error
	{
		driver drv({1, 1, false, false, false, 0});
		const auto devs = drv.devices();
		const rect vec({0}, {16});
		const auto a = drv.create_array(vec, dtype::f32, single_dist(vec, devs[0]), fill_spec::one());
		bool plan = false, parse = false;
		try {
			drv.launch("nope", vec, {4}, block_work_dist(vec, {4}, {16}, devs), {}, "global i =>");
		} catch(const plan_error&) {
			plan = true;
		}
		try {
			drv.launch("fill", vec, {4}, block_work_dist(vec, {4}, {16}, devs), {launch_arg::scalar(int64_t{16}), launch_arg::scalar(1.0), launch_arg::array(a)},
			    "global i => write out[i*i]");
		} catch(const parse_error&) {
			parse = true;
		}
		CHECK(plan && parse);
	}
	std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
	return failures ? 1 : 0;
}
