// Shared plumbing for the C ABI translation units.
#pragma once

#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/disc_b200.h"
#include "host/compiler.hpp"

namespace disc::rt {
struct PreparedPlan;  // device-side lowering of a plan's kernels (runtime/prepare.hpp)
std::shared_ptr<const PreparedPlan> prepare_plan(const CompiledPlan& plan);
}  // namespace disc::rt

// An immutable compiled plan plus its (lazily built, shape-agnostic) device lowering.
struct disc_plan_s {
  explicit disc_plan_s(std::shared_ptr<const disc::CompiledPlan> p) : plan(std::move(p)), serial(next_serial()) {}
  std::shared_ptr<const disc::CompiledPlan> plan;
  uint64_t serial;  // unique per plan object: keys executor launch caches
  static uint64_t next_serial() {
    static std::atomic<uint64_t> n{1};
    return n.fetch_add(1);
  }
  std::atomic<int> refs{1};
  std::once_flag prepared_once;
  std::shared_ptr<const disc::rt::PreparedPlan> prepared;
  const disc::rt::PreparedPlan& prep() {
    std::call_once(prepared_once, [&] { prepared = disc::rt::prepare_plan(*plan); });
    return *prepared;
  }
};

namespace disc_capi {
extern thread_local std::string g_error;
extern thread_local int g_error_class;
char* dup(const std::string& s);

// Runs f, mapping exceptions to the reference CLI's status codes (disc_main.cpp:353-366).
template <typename F>
int guard(F&& f) {
  try {
    f();
    g_error_class = -1;
    return 0;
  } catch (const disc::Error& e) {
    g_error = std::string("error[") + disc::error_class_name(e.error_class()) + "]: " + e.what();
    g_error_class = static_cast<int>(e.error_class());
    switch (e.error_class()) {
      case disc::ErrorClass::kUsage: return 2;
      case disc::ErrorClass::kParse:
      case disc::ErrorClass::kValidation:
      case disc::ErrorClass::kCompile: return 3;
      default: return 4;
    }
  } catch (const std::exception& e) {
    g_error = std::string("error[internal]: ") + e.what();
    g_error_class = static_cast<int>(disc::ErrorClass::kInternal);
    return 4;
  }
}

// EvalShape semantics (executor.cpp:303-341) for caller-provided input dims.
std::vector<int64_t> eval_shape_program(const disc::CompiledPlan& plan,
                                        const std::vector<std::vector<int64_t>>& input_dims);
}  // namespace disc_capi
