// store.h — device-resident CoefficientStore (see store.cu)
#pragma once

#include <cstddef>
#include <cuda_runtime.h>
#include <memory>

namespace qapb {

size_t store_nb(int m);
size_t store_nc(int m);
size_t store_nd(int m);

// b, c, d in the reference layout (StoreIndex, rlt2.hpp:25-69), in HBM
struct DeviceStore {
  int m = 0;
  int device = 0;
  double* b = nullptr;
  double* c = nullptr;
  double* d = nullptr;
  double offset = 0.0;
  cudaStream_t stream = nullptr;  // the store's own stream; arrays from the stream-ordered pool
  DeviceStore(int m_, int device_);
  ~DeviceStore();
  DeviceStore(const DeviceStore&) = delete;
  DeviceStore& operator=(const DeviceStore&) = delete;
  void synchronize() const;
};

// collapse_store, rlt2.cpp:109-182, bitwise, on the store's device
std::unique_ptr<DeviceStore> collapse_store_device(const DeviceStore& s, int fac, int loc);
// the same with the parent's constant term given (the child's is offset + b[fac, loc])
std::unique_ptr<DeviceStore> collapse_store_device(const DeviceStore& s, int fac, int loc,
                                                   double offset);
// store_evaluate, rlt2.cpp:91-107, bitwise (terms in the reference's order)
double store_evaluate_device(const DeviceStore& s, const int* perm, double offset);
// redistribute_family, rlt2.cpp:184-205
bool redistribute_family_device(const double pi[3], double add[3], int virtual_slots, double tol,
                                int device);

}  // namespace qapb
